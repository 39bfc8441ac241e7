# scratch GPU call used during round 2 (edited per call)
set -x
o=gpurun_out; tag=r2i
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke_$tag.txt 2>&1; echo smoke=$?
timeout 900 python bench.py > $o/bench_$tag.json 2> $o/bench_$tag.err; echo bench=$?
