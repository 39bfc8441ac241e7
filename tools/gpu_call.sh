# scratch GPU call used during round 2 (edited per call)
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_r2l.txt 2>&1; echo pytest=$?
tail -3 gpurun_out/gputest_r2l.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2l.txt 2>&1; echo smoke=$?
