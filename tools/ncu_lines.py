"""Per-source-line instruction counts and stall samples of one kernel from an ncu report
captured with --import-source on (run here, no GPU needed).

    python tools/ncu_lines.py gpurun_out/kga_src.ncu-rep [--top 40]
"""
import argparse
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=40)
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    f, rows = None, []
    hdr = None
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] in ("", "Function Name"):
            continue
        d = dict(zip(hdr[2:], r[2:]))
        try:
            inst = int(d["Instructions Executed"])
            samp = int(d["Warp Stall Sampling (All Samples)"])
        except (KeyError, ValueError):
            continue
        rows.append((inst, samp, f, r[0], r[1][:90]))
    tot_i = sum(x[0] for x in rows) or 1
    tot_s = sum(x[1] for x in rows) or 1
    print(f"total warp instructions {tot_i}, stall samples {tot_s}")
    for inst, samp, f, ln, src in sorted(rows, reverse=True)[:a.top]:
        print(f"{100*inst/tot_i:5.1f}% inst {100*samp/tot_s:5.1f}% samp  {f}:{ln}  {src}")


if __name__ == "__main__":
    main()
