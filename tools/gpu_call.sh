# scratch GPU call used during round 2 (edited per call)
sed -i 's/population=1 << 22/population=1 << 23/' tools/variant_bench.py
AB_WORKLOADS="TXT MIX" timeout 1200 bash tools/ab_run.sh gpurun_out/ab_tsec.jsonl build_variants/cur/libsaturn.so build_variants/tsec/libsaturn.so
tail -3 gpurun_out/ab_tsec.jsonl.err
python - <<'PY'
import json
for l in open('gpurun_out/ab_tsec.jsonl'):
    d=json.loads(l); print(d['lib'][:22], d['workload'], 'eval %.4g' % d['evaluate_plans_per_s'], 'step %.4f' % d['step_ms'], 'kga %.4f' % d['ga_kernel_ms'], d['best'])
PY
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:k_ga --launch-skip 6 --launch-count 1 python tools/variant_bench.py build_variants/tsec/libsaturn.so TXT 2>&1 | grep -E "dram__|gpu__time" 
