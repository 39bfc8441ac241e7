# scratch GPU call used during round 2 (edited per call)
set -x
o=gpurun_out; tag=r2h
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke_$tag.txt 2>&1; echo smoke=$?
timeout 900 python bench.py > $o/bench_$tag.json 2> $o/bench_$tag.err; echo bench=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/launches_$tag.csv \
  python bench.py --steps 3 --warmup 1 --no-cpu-baseline --kernel-only-n 0 > /dev/null 2>> $o/bench_$tag.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_ga --launch-skip 20 --launch-count 1 \
  -o $o/prof_ga_$tag python bench.py --steps 2 --warmup 1 --no-cpu-baseline --kernel-only-n 0 > /dev/null 2>> $o/bench_$tag.err
python tools/ncu_lines.py $o/prof_ga_$tag.ncu-rep > $o/k_ga_source_lines_$tag.txt 2>&1 || true
du -sh $o
