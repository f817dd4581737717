"""Phase breakdown of one traced factorization launch (SLIM_CHOL_TRACE csv).

t0 task start, t1 updates combined (MMA phase done), t2 diagonal ready /
POTRF done, t3 task end.  Prints per-kind mean phase times and the SM-slot
occupancy of the launch.
"""
import sys

import numpy as np

d = np.genfromtxt(sys.argv[1], delimiter=",", names=True, dtype=None, encoding=None)
t0, t1, t2, t3 = (d[f"t{q}"].astype(np.float64) for q in range(4))
ok = (t0 > 0) & (t3 > 0)
t0, t1, t2, t3 = t0[ok], t1[ok], t2[ok], t3[ok]
i, j, sysid = d["i"][ok], d["j"][ok], d["sys"][ok]
dual = (j & 0x8000) != 0
jj = j & 0x7FFF
kind = np.where(i == jj, "pair", np.where(dual, "dual", "single"))
base = t0.min()
span = (t3.max() - base) / 1e3
print(f"launch span {span:.1f} us, tasks {len(t0)}, mean task {np.mean(t3 - t0) / 1e3:.2f} us, "
      f"slot occupancy {np.sum(t3 - t0) / 1e3 / span / 148:.2f} CTAs/SM")
for k in ("pair", "dual", "single"):
    m = kind == k
    if not m.any():
        continue
    extra = ""
    if "slice_ns" in d.dtype.names:
        extra += (f"  [finish: slicing {np.mean(d['slice_ns'][ok][m]) / 1e3:5.2f} us, stores+publish "
                  f"{np.mean(d['store_ns'][ok][m]) / 1e3:5.2f} us]")
    if "dep_ns" in d.dtype.names:
        extra = (f"  [producer: dep wait {np.mean(d['dep_ns'][ok][m]) / 1e3:6.2f} us, MMA waits for data "
                 f"{np.mean(d['ring_ns'][ok][m]) / 1e3:6.2f} us]")
    print(f"{k:6s} n={m.sum():5d} k-tiles {np.mean(jj[m]):5.1f}  mma+combine {np.mean(t1[m] - t0[m]) / 1e3:6.2f} us"
          f"  wait/potrf {np.mean(t2[m] - t1[m]) / 1e3:6.2f}  finish {np.mean(t3[m] - t2[m]) / 1e3:6.2f}"
          f"  per k-tile {np.sum(t1[m] - t0[m]) / max(1, np.sum(jj[m])) / 1e3:.3f} us" + extra)
# time per k-tile for long tasks only (steady streaming)
m = (kind == "dual") & (jj >= 16)
if m.any():
    print(f"dual, >=16 k-tiles: {np.sum(t1[m] - t0[m]) / np.sum(jj[m]) / 1e3:.3f} us per k-tile")
