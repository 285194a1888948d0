"""Offline (CPU) replica of the resident kernel's CTA partition, to study
per-CTA balance (tuning aid). Mirrors vfpi_setup.cu phase 1."""
import sys

import numpy as np
import scipy.sparse as sp

sys.path.insert(0, ".")
from paper_2201_09212_b200.scenes import rigid_contact_system  # noqa: E402

EC, RC, CC = 24, 40, 256


def partition(ps, G=148, anchor=True, ec=EC, rc=RC, cc=CC):
    n = ps.n
    a = sp.csc_matrix((ps.data, ps.indices, ps.indptr), shape=(n, n)).tocsr()
    a.eliminate_zeros()
    rowcnt = np.diff(a.indptr)
    rowmin = np.array([a.indices[a.indptr[i]] if rowcnt[i] else n for i in range(n)])
    mark = -np.ones(n, int)
    for m, (i, j) in enumerate(zip(ps.col_i, ps.col_j)):
        mark[i:i + 3] = m
        if j >= 0:
            mark[j:j + 3] = m
    starts, keys = [], []
    for r in range(n):
        m = mark[r]
        if m < 0:
            starts.append(r); keys.append(min(r, rowmin[r]))
        elif r == ps.col_i[m]:
            i, j = ps.col_i[m], ps.col_j[m]
            rows = list(range(i, i + 3)) + (list(range(j, j + 3)) if j >= 0 else [])
            starts.append(r); keys.append(min(min(rows), min(rowmin[q] for q in rows)))
    starts = np.array(starts)
    order = np.argsort(np.array(keys), kind="stable") if anchor else np.arange(len(starts))
    U = starts[order]
    units = []
    for r in U:
        m = mark[r]
        if m < 0:
            units.append(([r], -1))
        else:
            i, j = ps.col_i[m], ps.col_j[m]
            units.append((list(range(i, i + 3)) + (list(range(j, j + 3)) if j >= 0 else []), m))
    cost = np.array([sum(ec * rowcnt[q] + rc for q in rows) + (cc if m >= 0 else 0) for rows, m in units])
    cpos = np.cumsum(cost) - cost
    blk = np.minimum(G - 1, cpos * G // cost.sum())
    ctas = []
    for b in range(G):
        us = [units[t] for t in np.nonzero(blk == b)[0]]
        crows = [q for rows, m in us if m >= 0 for q in rows]
        frows = sorted([rows[0] for rows, m in us if m < 0], key=lambda q: -rowcnt[q])
        rows = crows + frows
        own = set(rows)
        secs = set()
        for q in rows:
            for c in a.indices[a.indptr[q]:a.indptr[q + 1]]:
                if c not in own:
                    secs.add(c >> 2)
        lens = np.array([rowcnt[q] for q in rows])
        pad = np.pad(lens, (0, (-len(lens)) % 32)).reshape(-1, 32).max(1).sum() * 32 if len(lens) else 0
        ctas.append(dict(C=sum(1 for _, m in us if m >= 0), CR=len(crows), FR=len(frows), E=int(lens.sum()), EP=int(pad),
                         NS=len(secs), maxfree=int(max((rowcnt[q] for q in frows), default=0))))
    return ctas


if __name__ == "__main__":
    ps = rigid_contact_system(4096, 16384, 2201)
    for anchor in (False, True):
        ct = partition(ps, anchor=anchor)
        keys = ["C", "CR", "FR", "E", "EP", "NS", "maxfree"]
        print("anchor" if anchor else "natural")
        for k in keys:
            v = np.array([c[k] for c in ct])
            print(f"  {k:8s} mean {v.mean():8.1f} max {v.max():6d} min {v.min():6d}")
