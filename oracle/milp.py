"""O4b: the paper's SPASE MILP (Eqs. 1-11) solved by HiGHS.

TEST INFRASTRUCTURE ONLY (also the f3 "MILP bar": the paper's own method with an
open-source solver in place of Gurobi).

Variables (Table 1): B[t,s], O[t,n], P[t,n,g], A[t1,t2] binary;
I[t,n,g] >= 0 and C >= 0 continuous.  Big-M U = H + max_n GPU_n + 1 with
H = sum_t max_s R_{t,s}.  Constraint rows, with the readings listed in
DESIGN.md:

  Eq. 2  C >= I[t,n,g] + R[t,s] - U(1 - B[t,s])      all t, s, n, g in GPU_n (A3)
  Eq. 3  sum_s B[t,s] = 1 ; sum_n O[t,n] = 1
  Eq. 4  sum_g P[t,n,g] >= G[t,s] - U(2 - O[t,n] - B[t,s])
  Eq. 5  sum_g P[t,n,g] <= G[t,s] + U(2 - O[t,n] - B[t,s])
  Eq. 6-7 (A1; prose PAPER.md:865)  sum_g P[t,n,g] <= U O[t,n]      (printed form is infeasible)
  Eq. 8  sum_x I[t,n,x] / G[t,s] <= I[t,n,g] + U(3 - P[t,n,g] - B[t,s] - O[t,n])
  Eq. 9  sum_x I[t,n,x] / G[t,s] >= I[t,n,g] - U(3 - P[t,n,g] - B[t,s] - O[t,n])
  Eq. 10 (A2 binds t = t1)
         I[t1,n,g] <= I[t2,n,g] - R[t1,s] + U((3 - P[t1,n,g] - P[t2,n,g]) - B[t1,s] + A[t2,t1])
  Eq. 11 (A2 binds t = t2)
         I[t1,n,g] >= I[t2,n,g] + R[t2,s] - U((4 - P[t1,n,g] - P[t2,n,g]) - A[t2,t1] - B[t2,s])
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
from scipy.optimize import Bounds, LinearConstraint, milp


class SpaseMilp:
    def __init__(self, c):
        self.c = c
        T = c.n_jobs
        N = len(c.node_gpus)
        self.T, self.N = T, N
        gpus = [int(x) for x in c.node_gpus]
        H = sum(max(c.config(t, s)[2] for s in range(int(c.S[t]))) for t in range(T))
        self.U = U = float(H + max(gpus) + 1)
        idx = {}
        kinds = []

        def var(key, integer):
            idx[key] = len(kinds)
            kinds.append(integer)

        for t in range(T):
            for s in range(int(c.S[t])):
                var(("B", t, s), 1)
        for t in range(T):
            for n in range(N):
                var(("O", t, n), 1)
        for t in range(T):
            for n in range(N):
                for g in range(gpus[n]):
                    var(("P", t, n, g), 1)
        for t1 in range(T):
            for t2 in range(T):
                if t1 != t2:
                    var(("A", t1, t2), 1)
        for t in range(T):
            for n in range(N):
                for g in range(gpus[n]):
                    var(("I", t, n, g), 0)
        var(("C",), 0)
        self.idx, self.kinds = idx, np.array(kinds)
        nv = len(kinds)

        rows, cols, vals, lo, hi, tags = [], [], [], [], [], []

        def row(terms, l, h, tag):
            r = len(lo)
            for k, v in terms:
                rows.append(r)
                cols.append(idx[k])
                vals.append(v)
            lo.append(l)
            hi.append(h)
            tags.append(tag)

        inf = np.inf
        G = lambda t, s: c.config(t, s)[1]     # noqa: E731
        R = lambda t, s: c.config(t, s)[2]     # noqa: E731
        for t in range(T):                     # Eq. 2
            for s in range(int(c.S[t])):
                for n in range(N):
                    for g in range(gpus[n]):
                        row([(("C",), 1), (("I", t, n, g), -1), (("B", t, s), -U)], R(t, s) - U, inf, "makespan")
        for t in range(T):                     # Eq. 3
            row([(("B", t, s), 1) for s in range(int(c.S[t]))], 1, 1, "one-config")
            row([(("O", t, n), 1) for n in range(N)], 1, 1, "one-node")
        for t in range(T):                     # Eqs. 4-5
            for s in range(int(c.S[t])):
                for n in range(N):
                    P = [(("P", t, n, g), 1) for g in range(gpus[n])]
                    row(P + [(("O", t, n), -U), (("B", t, s), -U)], G(t, s) - 2 * U, inf, "alloc-lo")
                    row(P + [(("O", t, n), U), (("B", t, s), U)], -inf, G(t, s) + 2 * U, "alloc-hi")
        for t in range(T):                     # Eqs. 6-7, reading A1
            for n in range(N):
                row([(("P", t, n, g), 1) for g in range(gpus[n])] + [(("O", t, n), -U)], -inf, 0, "unselected-zero")
        for t in range(T):                     # Eqs. 8-9
            for s in range(int(c.S[t])):
                for n in range(N):
                    for g in range(gpus[n]):
                        avg = [(("I", t, n, x), 1.0 / G(t, s)) for x in range(gpus[n])]
                        ind = [(("P", t, n, g), U), (("B", t, s), U), (("O", t, n), U)]
                        # avg - I_g + U P + U B + U O <= 3U   (x in avg may equal g: coefficients add)
                        row(avg + [(("I", t, n, g), -1)] + ind, -inf, 3 * U, "gang-lo")
                        row(avg + [(("I", t, n, g), -1)] + [(k, -v) for k, v in ind], -3 * U, inf, "gang-hi")
        for t1 in range(T):                    # Eqs. 10-11
            for t2 in range(T):
                if t1 == t2:
                    continue
                for n in range(N):
                    for g in range(gpus[n]):
                        base = [(("I", t1, n, g), 1), (("I", t2, n, g), -1)]
                        for s in range(int(c.S[t1])):   # Eq. 10 binds t = t1
                            row(base + [(("P", t1, n, g), U), (("P", t2, n, g), U), (("B", t1, s), U),
                                        (("A", t2, t1), -U)], -inf, 3 * U - R(t1, s), "isolation-before")
                        for s in range(int(c.S[t2])):   # Eq. 11 binds t = t2
                            row(base + [(("P", t1, n, g), -U), (("P", t2, n, g), -U), (("A", t2, t1), -U),
                                        (("B", t2, s), -U)], R(t2, s) - 4 * U, inf, "isolation-after")
        self.A = sp.csr_matrix((vals, (rows, cols)), shape=(len(lo), nv))  # duplicates are summed
        self.lo, self.hi, self.tags = np.array(lo), np.array(hi), tags
        ub = np.where(self.kinds == 1, 1.0, np.inf)
        self.bounds = Bounds(np.zeros(nv), ub)
        self.obj = np.zeros(nv)
        self.obj[idx[("C",)]] = 1.0

    @property
    def n_vars(self) -> int:
        return self.A.shape[1]

    @property
    def n_rows(self) -> int:
        return self.A.shape[0]

    def solve(self, time_limit: float = 60.0):
        """-> (status, makespan or None, plan or None).  status: 'optimal' | 'incumbent' | 'none'."""
        res = milp(self.obj, constraints=LinearConstraint(self.A, self.lo, self.hi), integrality=self.kinds,
                   bounds=self.bounds, options={"time_limit": time_limit, "mip_rel_gap": 0.0, "disp": False})
        if res.x is None:
            return "none", None, None
        status = "optimal" if res.status == 0 else "incumbent"
        return status, float(res.fun), self.solution_to_plan(res.x)

    def violations(self, x, tol: float = 1e-6):
        """check_solution: tags of violated rows plus non-integral binaries."""
        ax = self.A @ x
        bad = [self.tags[i] for i in np.nonzero((ax < self.lo - tol) | (ax > self.hi + tol))[0]]
        ints = x[self.kinds == 1]
        if np.any(np.abs(ints - np.round(ints)) > tol):
            bad.append("integrality")
        return bad

    def plan_to_assignment(self, placements, makespan):
        """Plan -> 0/1/continuous assignment of B, O, P, A, I, C (round trip of SPEC.md:192)."""
        c, x = self.c, np.zeros(self.n_vars)
        for t, pl in enumerate(placements):
            x[self.idx[("B", t, pl["cfg"])]] = 1
            x[self.idx[("O", t, pl["node"])]] = 1
            for g in range(int(c.node_gpus[pl["node"]])):
                if pl["gpu_mask"] >> g & 1:
                    x[self.idx[("P", t, pl["node"], g)]] = 1
                    x[self.idx[("I", t, pl["node"], g)]] = pl["start_s"]
        for t1 in range(self.T):
            for t2 in range(self.T):
                if t1 != t2:
                    # A[t1,t2] = 1 iff t1 runs before t2 (Table 1); order by start, then job id
                    a, b = placements[t1], placements[t2]
                    x[self.idx[("A", t1, t2)]] = 1 if (a["start_s"], t1) < (b["start_s"], t2) else 0
        x[self.idx[("C",)]] = makespan
        return x

    # ---------------------------------------------------------------- LP export (row f3)
    def var_name(self, key) -> str:
        """B_t_s, O_t_n, P_t_n_g, A_t1_t2, I_t_n_g, C (Table 1's symbols)."""
        return "_".join(str(k) for k in key)

    def to_lp(self, f) -> None:
        """Write the MILP in CPLEX LP format (the format PuLP hands to Gurobi/CBC):
        objective, one named row per constraint (tag_index; ranged rows as two), bounds,
        binaries.  `f` is a path or a text file object."""
        if isinstance(f, str):
            with open(f, "w") as fh:
                return self.to_lp(fh)
        names = [None] * self.n_vars
        for key, j in self.idx.items():
            names[j] = self.var_name(key)

        def fmt(v):
            return repr(float(v)) if not float(v).is_integer() else str(int(v))

        def lin(r):
            a, b = self.A.indptr[r], self.A.indptr[r + 1]
            parts = []
            for j, v in zip(self.A.indices[a:b], self.A.data[a:b]):
                if v == 0:
                    continue
                parts.append(("- " if v < 0 else "+ ") + fmt(abs(v)) + " " + names[j])
            return " ".join(parts) if parts else "0 C"

        f.write("\\ SPASE MILP, PAPER.md Eqs. 1-11 (readings A1-A3, DESIGN.md)\n")
        f.write(f"Minimize\n obj: {names[self.idx[('C',)]]}\nSubject To\n")
        for r in range(self.n_rows):
            lo, hi, e = self.lo[r], self.hi[r], lin(r)
            tag = f"{self.tags[r].replace('-', '_')}_{r}"
            if lo == hi:
                f.write(f" {tag}: {e} = {fmt(lo)}\n")
            else:
                if np.isfinite(lo):
                    f.write(f" {tag}_lo: {e} >= {fmt(lo)}\n")
                if np.isfinite(hi):
                    f.write(f" {tag}_hi: {e} <= {fmt(hi)}\n")
        f.write("Bounds\n")
        for j in range(self.n_vars):
            if self.kinds[j] == 0:
                f.write(f" {names[j]} >= 0\n")
        f.write("Binaries\n")
        for j in range(self.n_vars):
            if self.kinds[j] == 1:
                f.write(f" {names[j]}\n")
        f.write("End\n")

    def solution_to_plan(self, x):
        c, plan = self.c, []
        for t in range(self.T):
            s = max(range(int(c.S[t])), key=lambda s: x[self.idx[("B", t, s)]])
            n = max(range(self.N), key=lambda n: x[self.idx[("O", t, n)]])
            mask, start = 0, None
            for g in range(int(c.node_gpus[n])):
                if x[self.idx[("P", t, n, g)]] > 0.5:
                    mask |= 1 << g
                    start = x[self.idx[("I", t, n, g)]] if start is None else start
            _, gg, r = c.config(t, s)
            st = int(round(start or 0.0))
            plan.append(dict(node=n, upp=c.config(t, s)[0], gpus=gg, cfg=s, start_s=st, end_s=st + r,
                             gpu_mask=mask))
        return plan


def read_lp(text: str):
    """Minimal reader of the LP files to_lp writes (for the round-trip pin): -> (objective
    variable, {row name: ({var: coef}, sense, rhs)}, binaries, nonnegatives)."""
    sec, rows, binaries, nonneg, obj = None, {}, [], [], None
    for raw in text.splitlines():
        ln = raw.strip()
        if not ln or ln.startswith("\\"):
            continue
        if ln in ("Minimize", "Subject To", "Bounds", "Binaries", "End"):
            sec = ln
            continue
        if sec == "Minimize":
            obj = ln.split(":", 1)[1].strip()
        elif sec == "Subject To":
            name, rest = ln.split(":", 1)
            for op in (">=", "<=", "="):
                if f" {op} " in rest:
                    lhs, rhs = rest.rsplit(f" {op} ", 1)
                    break
            toks, coef = lhs.split(), {}
            for k in range(0, len(toks), 3):
                sign, val, var = toks[k], float(toks[k + 1]), toks[k + 2]
                coef[var] = coef.get(var, 0.0) + (val if sign == "+" else -val)
            rows[name.strip()] = (coef, op, float(rhs))
        elif sec == "Bounds":
            nonneg.append(ln.split()[0])
        elif sec == "Binaries":
            binaries.append(ln)
    return obj, rows, binaries, nonneg


def milp_makespan(c, time_limit: float = 60.0):
    m = SpaseMilp(c)
    status, val, plan = m.solve(time_limit)
    return status, (None if val is None else int(round(val))), plan
