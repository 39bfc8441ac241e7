"""Instruction mix of the loops of one kernel in a cubin (static SASS, run here):
    python tools/sass_loops.py <cubin> <kernel-name-substring> [min_len]
Prints each backward-branch loop body with its opcode counts and the ALU / FMA-pipe split."""
import collections
import re
import subprocess
import sys

ALU = {"SEL", "VIMNMX", "ISETP", "LOP3", "SHF", "IADD3", "LEA", "PRMT", "POPC", "FLO", "PLOP3", "VIADD", "IMNMX",
       "MOV", "BREV"}
FMA = {"IMAD", "IMUL", "FFMA", "FMUL", "FADD"}


def main():
    cubin, name = sys.argv[1], sys.argv[2]
    min_len = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    txt = subprocess.run(["nvdisasm", cubin], capture_output=True, text=True).stdout
    secs = re.split(r"\n\s*\.section\s+\.text\.", txt)
    sec = next(s for s in secs if s.split(",")[0].find(name) >= 0)
    lab, cur, addr, ins = {}, None, [], []
    for l in sec.splitlines():
        m = re.match(r"^(\.L_x_\d+):", l.strip())
        if m:
            cur = m.group(1)
            continue
        m = re.search(r"/\*([0-9a-f]{4,5})\*/\s*(.*?);", l)
        if m:
            a = int(m.group(1), 16)
            if cur:
                lab[cur] = a
                cur = None
            addr.append(a)
            ins.append(m.group(2).strip())
    for i, t in enumerate(ins):
        m = re.search(r"BRA.*?`\((\.L_x_\d+)\)", t)
        if not m or m.group(1) not in lab or lab[m.group(1)] >= addr[i]:
            continue
        body = [ins[k] for k in range(len(ins)) if lab[m.group(1)] <= addr[k] <= addr[i]]
        if len(body) < min_len:
            continue
        ops = collections.Counter()
        for x in body:
            tok = x.split()
            op = tok[1] if tok[0].startswith("@") else tok[0]
            ops[op.split(".")[0]] += 1
        alu = sum(v for k, v in ops.items() if k in ALU)
        fma = sum(v for k, v in ops.items() if k in FMA)
        print(f"{hex(addr[i])}: {len(body)} instr, ALU {alu}, FMA {fma}, other {len(body) - alu - fma}: "
              f"{dict(ops.most_common(10))}")


if __name__ == "__main__":
    main()
