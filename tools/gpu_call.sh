# scratch GPU call used during round 2 (edited per call)
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_r2j.txt 2>&1; echo pytest=$?; tail -2 gpurun_out/gputest_r2j.txt
