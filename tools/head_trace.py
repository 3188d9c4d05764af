"""Summarise the head kernel's timeline probe (SC_HEAD_TRACE=file, see trace_slot in sc_head.cu).

usage: python tools/head_trace.py TRACE.bin
Takes the last launch's record: [8 CTAs][32 units][16 slots] uint64 (ns / summed ns)."""
import sys

import numpy as np

CTAS, UNITS, SLOTS = 8, 32, 16
a = np.fromfile(sys.argv[1], dtype=np.uint64)
n = CTAS * UNITS * SLOTS
rec = a[-n:].reshape(CTAS, UNITS, SLOTS).astype(np.int64)
print(f"{len(a) // n} launches recorded; the last one (steady-state units 2..29):")
rows = []
for c in range(CTAS):
    r = rec[c]
    valid = r[:, 1] > 0
    u = np.nonzero(valid)[0]
    if len(u) == 0:  # a CTA pair's second CTA: no MMA issuer
        continue
    u = u[(u >= 2) & (u < u.max())]
    if len(u) < 2:
        continue
    period = np.diff(r[u, 1]).mean()
    rows.append(dict(
        period=period,
        mma_wait_acc=(r[u, 1] - r[u, 0]).mean(),
        mma_wait_x=r[u, 2].mean(), mma_wait_w=r[u, 3].mean(),
        mma_issue=(r[u, 4] - r[u, 1]).mean(),
        epi_wait=(r[u, 6] - r[u, 5]).mean(), epi_drain=(r[u, 7] - r[u, 6]).mean(),
        epi_finish=(r[u, 8] - r[u, 7]).mean(),
        epi7_drain=(r[u, 12] - r[u, 11]).mean(),
        acc_ready_to_drain_start=(r[u, 6] - r[u, 4]).mean(),
        xprod_wait=r[u, 9].mean(), wprod_wait=r[u, 10].mean()))
# CTAs without an MMA issuer (a pair's second CTA): their producers' and epilogue's numbers
for c in range(CTAS):
    r = rec[c]
    if (r[:, 1] > 0).any() or not (r[:, 6] > 0).any():
        continue
    u = np.arange(2, UNITS - 1)
    print(f"CTA {c} (pair peer): epi_wait {(r[u, 6] - r[u, 5]).mean() / 1e3:.2f}  epi_drain "
          f"{(r[u, 7] - r[u, 6]).mean() / 1e3:.2f}  epi_finish {(r[u, 8] - r[u, 7]).mean() / 1e3:.2f}  "
          f"xprod_wait {r[u, 9].mean() / 1e3:.2f}  wprod_wait {r[u, 10].mean() / 1e3:.2f} (us)")
keys = list(rows[0].keys())
print("CTA  " + "  ".join(f"{k:>12s}" for k in keys))
for c, d in enumerate(rows):
    print(f"{c:3d}  " + "  ".join(f"{d[k] / 1e3:12.2f}" for k in keys))
m = {k: np.mean([d[k] for d in rows]) / 1e3 for k in keys}
print("mean " + "  ".join(f"{m[k]:12.2f}" for k in keys), "(us)")
