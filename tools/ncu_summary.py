"""Summarise ncu captures and launch lists into profiles/<round>/ (run here, no GPU needed).

    python tools/ncu_summary.py --round r1 --ga gpurun_out/prof_ga_r1g.ncu-rep \
        --eval gpurun_out/prof_eval_r1g.ncu-rep --launches gpurun_out/launches_r1g.csv
"""
from __future__ import annotations

import argparse
import collections
import csv
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'sm__cycles_elapsed.avg.per_second', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'dram__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread', 'launch__grid_size',
        'launch__block_size', 'smsp__inst_executed.sum', 'smsp__sass_inst_executed_op_local_ld.sum',
        'smsp__sass_inst_executed_op_local_st.sum', 'smsp__inst_executed_pipe_uniform.sum']
STALLS = 'smsp__pcsamp_warps_issue_stalled_'
SCALE = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}


def raw(rep):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))


def summarise(rep):
    d, u = raw(rep)
    out = {k: [d[k], u.get(k, '')] for k in KEYS if k in d}
    st = {k[len(STALLS):]: float(d[k] or 0) for k in d if k.startswith(STALLS) and not k.endswith('not_issued')}
    tot = sum(st.values()) or 1.0
    out['stall_share'] = {k: round(v / tot, 3) for k, v in sorted(st.items(), key=lambda x: -x[1])[:8]}
    num = lambda k: float(d[k].replace(',', '')) * SCALE.get(u[k], 1)  # noqa: E731
    out['dram_bytes_per_launch'] = int(num('dram__bytes_read.sum') + num('dram__bytes_write.sum'))
    return out


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
    h = rows[hi]
    ki, vi = h.index('Kernel Name'), h.index('Metric Value')
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split('(')[0].replace('void ', '').split('<')[0]
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(',', ''))
    tot = sum(v[1] for v in agg.values())
    return {k: {"launches": n, "avg_us": t / n / 1e3, "share": t / tot} for k, (n, t) in
            sorted(agg.items(), key=lambda x: -x[1][1])}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument('--round', default='r1')
    ap.add_argument('--ga')
    ap.add_argument('--eval')
    ap.add_argument('--launches')
    ap.add_argument('--enum')
    ap.add_argument('--sweep', help='k_ga capture at the SWEEP workload (tools/variant_bench.py)')
    ap.add_argument('--workload', default='TXT')
    ap.add_argument('--merge', action='store_true', help='update the existing summary instead of replacing it')
    args = ap.parse_args()
    outdir = os.path.join(ROOT, 'profiles', args.round)
    os.makedirs(outdir, exist_ok=True)
    path = os.path.join(outdir, 'ncu_summary.json')
    summ = json.load(open(path)) if args.merge and os.path.exists(path) else {}
    if args.ga:
        summ['k_ga (bench config)'] = summarise(args.ga)
        with open(os.path.join(ROOT, 'profiles', 'roofline_traffic.json'), 'w') as f:
            json.dump({"_about": "dram__bytes_read.sum + dram__bytes_write.sum of one k_ga launch at bench.py's "
                                 "default config, from one ncu --set full capture (profiles/%s/ncu_summary.json)"
                                 % args.round, args.workload: summ['k_ga (bench config)']['dram_bytes_per_launch']},
                      f, indent=1)
    if args.eval:
        summ['k_evaluate (2^24 genomes)'] = summarise(args.eval)
    if args.enum:
        summ['k_enumerate (TINY-shaped 7 jobs, 1.41e9 genomes)'] = summarise(args.enum)
    if args.sweep:
        summ['k_ga (SWEEP 4x8, 2^22 genomes, tools/variant_bench.py)'] = summarise(args.sweep)
    if args.launches:
        summ['launch_list_shares'] = launches(args.launches)
    with open(path, 'w') as f:
        json.dump(summ, f, indent=1)
    print(json.dumps(summ, indent=1))


if __name__ == '__main__':
    main()
