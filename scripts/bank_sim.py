"""Offline estimate of shared-memory wavefronts of the resident kernel's x
gathers on configs[1] (anchor order), current placement vs a bank-aware
placement of the staged sectors (tuning aid)."""
import sys

import numpy as np
import scipy.sparse as sp

sys.path.insert(0, ".")
from paper_2201_09212_b200.scenes import rigid_contact_system  # noqa: E402


def layout(ps, G=148, ec=24, rc=40):
    n = ps.n
    a = sp.csc_matrix((ps.data, ps.indices, ps.indptr), shape=(n, n)).tocsr()
    a.eliminate_zeros()
    a.sort_indices()
    rowcnt = np.diff(a.indptr)
    rowmin = np.array([a.indices[a.indptr[i]] if rowcnt[i] else n for i in range(n)])
    mark = -np.ones(n, int)
    for m, (i, j) in enumerate(zip(ps.col_i, ps.col_j)):
        mark[i:i + 3] = m
        if j >= 0:
            mark[j:j + 3] = m
    units = []
    for r in range(n):
        m = mark[r]
        if m < 0:
            units.append((min(r, rowmin[r]), [r], -1))
        elif r == ps.col_i[m]:
            i, j = ps.col_i[m], ps.col_j[m]
            rows = list(range(i, i + 3)) + (list(range(j, j + 3)) if j >= 0 else [])
            units.append((min(min(rows), min(rowmin[q] for q in rows)), rows, m))
    units.sort(key=lambda u: u[0])
    cost = np.array([sum(ec * rowcnt[q] + rc for q in rows) for _, rows, _ in units])
    cpos = np.cumsum(cost) - cost
    blk = np.minimum(G - 1, cpos * G // cost.sum())
    ctas = []
    for b in range(G):
        us = [units[t] for t in np.nonzero(blk == b)[0]]
        cs = [u for u in us if u[2] >= 0]
        C = len(cs)
        CD = sum(1 for u in cs if len(u[1]) == 6)
        crow = [None] * (3 * C + 3 * CD)
        kd = 0
        for k, (_, rows, m) in enumerate(cs):
            for t in range(3):
                crow[t * C + k] = rows[t]
            if len(rows) == 6:
                for t in range(3):
                    crow[3 * C + t * CD + kd] = rows[3 + t]
                kd += 1
        frows = sorted([u[1][0] for u in us if u[2] < 0], key=lambda q: -rowcnt[q])
        ctas.append(crow + frows)
    return a, ctas


def wavefronts(items):
    """items: list of (address, bank) of one warp request (distinct lanes)."""
    banks = {}
    for addr, bank in set(items):
        banks.setdefault(bank, set()).add(addr)
    if not banks:
        return 0
    distinct = sum(len(v) for v in banks.values())
    return max(max(len(v) for v in banks.values()), -(-distinct // 16))


def analyse(a, rows, greedy=False):
    pos = {r: q for q, r in enumerate(rows)}
    R = len(rows)
    cols = [a.indices[a.indptr[r]:a.indptr[r + 1]] for r in rows]
    secs = sorted({c >> 2 for cs in cols for c in cs if c not in pos})
    # warp-steps: (slice, k) -> list of x items (kind, key, off)
    steps = []
    for s0 in range(0, R, 32):
        W = max(len(cols[q]) for q in range(s0, min(s0 + 32, R)))
        for k in range(W):
            it = []
            for q in range(s0, min(s0 + 32, R)):
                if k < len(cols[q]):
                    c = cols[q][k]
                    it.append(("o", pos[c], 0) if c in pos else ("s", c >> 2, c & 3))
            steps.append(it)
    phase = {s: i % 4 for i, s in enumerate(secs)}
    own_bank = {q: q % 16 for q in range(R)}

    def bank(x):
        return own_bank[x[1]] if x[0] == "o" else (4 * phase[x[1]] + x[2]) % 16

    def total():
        return sum(wavefronts([((x[0], x[1], x[2]), bank(x)) for x in st]) for st in steps)

    base = total()
    if not greedy:
        return base, None
    # greedy: sectors by use count, phase minimising the bank load of their steps
    uses = {}
    for si, st in enumerate(steps):
        for x in st:
            if x[0] == "s":
                uses.setdefault(x[1], []).append(si)
    load = [dict() for _ in steps]  # bank -> set(addr)
    for si, st in enumerate(steps):
        for x in st:
            if x[0] == "o":
                load[si].setdefault(own_bank[x[1]], set()).add(x)
    for s in sorted(uses, key=lambda s: -len(uses[s])):
        best, bp = None, 0
        for ph in range(4):
            c = 0
            for si in uses[s]:
                for x in steps[si]:
                    if x[0] == "s" and x[1] == s:
                        b = (4 * ph + x[2]) % 16
                        c += len(load[si].get(b, ()))
            if best is None or c < best:
                best, bp = c, ph
        phase[s] = bp
        for si in uses[s]:
            for x in steps[si]:
                if x[0] == "s" and x[1] == s:
                    load[si].setdefault((4 * bp + x[2]) % 16, set()).add(x)
    return base, total()


if __name__ == "__main__":
    ps = rigid_contact_system(4096, 16384, 2201)
    a, ctas = layout(ps)
    for b in (0, 50, 100):
        ent = sum(np.diff(a.indptr)[ctas[b]])
        base, g = analyse(a, ctas[b], greedy=True)
        print(f"cta {b}: rows {len(ctas[b])} entries {ent} ideal(2/32 per entry) {2 * ent / 32:.0f} "
              f"wavefronts current {base} greedy-phase {g}")
