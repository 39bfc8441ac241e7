#!/bin/bash
# One GPU call that refreshes the round's evidence under gpurun_out/ (then run
# tools/ncu_summary.py here to write profiles/<round>/):
#   bench lines (TXT default + the other workloads), the ncu launch list of the bench
#   command, and one `ncu --set full` capture each of k_ga, k_evaluate and k_enumerate_dfs.
#   tools/profile_round.sh r1i
tag=${1:-r1}
o=gpurun_out
python bench.py > $o/bench_$tag.json 2> $o/bench_$tag.err
for w in IMG MIX SWEEP TINY; do
  python bench.py --workload $w --steps 20 --no-cpu-baseline > $o/bench_${tag}_$w.json 2>> $o/bench_$tag.err
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/launches_$tag.csv \
  python bench.py --steps 3 --warmup 1 --no-cpu-baseline --kernel-only-n 0 > /dev/null 2>> $o/bench_$tag.err
ncu --set full --import-source on --clock-control none -k regex:k_ga --launch-skip 20 --launch-count 1 \
  -o $o/prof_ga_$tag python bench.py --steps 2 --warmup 1 --no-cpu-baseline --kernel-only-n 0 > /dev/null 2>> $o/bench_$tag.err
ncu --set full --import-source on --clock-control none -k regex:k_evaluate --launch-count 1 \
  -o $o/prof_eval_$tag python tools/variant_bench.py paper_2309_01226_b200/libsaturn.so TXT > /dev/null 2>> $o/bench_$tag.err
ncu --set full --import-source on --clock-control none -k regex:k_enumerate_dfs --launch-count 1 \
  -o $o/prof_enum_$tag python tools/enum_once.py > /dev/null 2>> $o/bench_$tag.err
ls -la $o | tail -12
