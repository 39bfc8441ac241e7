# scratch GPU call used during round 2 (edited per call)
start=$(date +%s); python bench.py > gpurun_out/bench_r2a.json 2> gpurun_out/bench_r2a.err; echo "bench wall $(( $(date +%s) - start )) s"; tail -3 gpurun_out/bench_r2a.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_r2a.json').read().strip().splitlines()[-1])
print({k: d[k] for k in ('value','ms_per_step','clocks','gpu_launches')})
print('roofline', {k: d['roofline'][k] for k in ('frac','launch_ms','kernel_share_of_step')})
print('e2e', d['e2e'])
for k,v in (d['workloads'] or {}).items(): print(k, {kk: (round(vv,4) if isinstance(vv,float) else vv) for kk,vv in v.items() if kk!='workload'})
for q in d['quality'] or []: print({k:q[k] for k in ('workload','table_seed','best','cpu_5min_bar','beats_bar','lower_bound','wall_s')})
print(d['best_vs_oracle']); print(d['cpu_baseline']); print(d['host_cpu'])
PY
