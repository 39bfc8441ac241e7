# scratch GPU call used during round 2 (edited per call)
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_r2k.txt 2>&1; echo pytest=$?
tail -3 gpurun_out/gputest_r2k.txt
timeout 900 python bench.py > gpurun_out/bench_r2k.json 2> gpurun_out/bench_r2k.err; echo bench=$?
