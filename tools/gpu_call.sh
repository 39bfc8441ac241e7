# scratch GPU call used during round 2 (edited per call)
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
AB_WORKLOADS="TXT MIX SWEEP" timeout 1200 bash tools/ab_run.sh gpurun_out/ab_ahead.jsonl build_variants/prev/libsaturn.so build_variants/ahead2/libsaturn.so
tail -3 gpurun_out/ab_ahead.jsonl.err
python - <<'PY'
import json
for l in open('gpurun_out/ab_ahead.jsonl'):
    d=json.loads(l); print(d['lib'][:22], d['workload'], 'eval %.4g' % d['evaluate_plans_per_s'], 'step %.4f' % d['step_ms'], 'kga %.4f' % d['ga_kernel_ms'], d['best'])
PY
timeout 600 python tools/exp_lane_per_node.py --out gpurun_out/exp_lanes.json 2>&1 | tail -4
