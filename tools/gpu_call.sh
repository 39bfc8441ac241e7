# scratch GPU call used during round 2 (edited per call)
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_r2e.txt 2>&1; echo pytest=$?
tail -3 gpurun_out/gputest_r2e.txt
timeout 2400 bash tools/profile_round.sh r2e
python tools/ncu_lines.py gpurun_out/prof_ga_r2e.ncu-rep > gpurun_out/k_ga_source_lines_r2e.txt 2>&1 || true
