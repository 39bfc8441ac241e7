# scratch GPU call used during round 2 (edited per call)
set -x
o=gpurun_out; tag=r2g
timeout 1500 python -m pytest tests -m gpu -x -q > $o/gputest_$tag.txt 2>&1; echo pytest=$?
tail -3 $o/gputest_$tag.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke_$tag.txt 2>&1; echo smoke=$?
timeout 900 python bench.py > $o/bench_$tag.json 2> $o/bench_$tag.err; echo bench=$?
