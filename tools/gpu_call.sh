# scratch GPU call used during round 2 (edited per call)
set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_r2i.txt 2>&1; echo pytest=$?
tail -3 gpurun_out/gputest_r2i.txt
sed -i 's/population=1 << 22/population=1 << 23/' tools/variant_bench.py
AB_WORKLOADS="TXT MIX TINY" timeout 1500 bash tools/ab_run.sh gpurun_out/ab_ppf.jsonl build_variants/cur/libsaturn.so build_variants/noppf/libsaturn.so
tail -3 gpurun_out/ab_ppf.jsonl.err
python - <<'PY'
import json
for l in open('gpurun_out/ab_ppf.jsonl'):
    d=json.loads(l); print(d['lib'][-22:], d['workload'], 'eval %.4g' % d['evaluate_plans_per_s'], 'step %.4f' % d['step_ms'], 'kga %.4f' % d['ga_kernel_ms'], d['best'])
PY
