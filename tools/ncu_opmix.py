"""Executed-instruction mix of one kernel by SASS opcode and by pipe (from an ncu report
captured with --import-source on; run here, no GPU needed).

    python tools/ncu_opmix.py gpurun_out/prof_ga_v5.ncu-rep
"""
import collections
import csv
import io
import subprocess
import sys

# pipe of each opcode family on sm_100 (B300_MICROARCH.md "Pipe rates": IMAD/FFMA on the
# FMA pipe; IADD3/LOP3/SHF/PRMT/MNMX/SEL/ISETP on the ALU pipe)
FMA = {"IMAD", "FFMA", "FMUL", "FADD", "HFMA2", "IMUL"}
ALU = {"IADD3", "LOP3", "SHF", "PRMT", "VIMNMX", "IMNMX", "FMNMX", "SEL", "ISETP", "LEA", "R2P", "P2R", "VIADD",
       "IABS", "FSEL", "FSETP", "PLOP3", "MOV", "LOP", "BMSK", "FLO", "POPC", "BREV", "IADD"}


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ix, ie = hdr.index("Source"), hdr.index("Instructions Executed")
    ops = collections.Counter()
    for r in rows[2:]:
        if len(r) <= ie or not r[ie].isdigit():
            continue
        src = r[ix].strip()
        if src.startswith("@"):
            src = src.split(None, 1)[1]
        op = src.split()[0].rstrip(";")
        ops[op] += int(r[ie])
    tot = sum(ops.values())
    pipes = collections.Counter()
    for op, n in ops.items():
        base = op.split(".")[0]
        pipes["fma" if base in FMA else "alu" if base in ALU else "lsu/other:" + base] += n
    print(f"total warp instructions {tot}")
    for p, n in sorted(pipes.items(), key=lambda x: -x[1])[:20]:
        print(f"  {p:24s} {100 * n / tot:5.1f}%")
    for op, n in ops.most_common(30):
        print(f"  {op:28s} {100 * n / tot:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
