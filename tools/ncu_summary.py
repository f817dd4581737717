"""Summaries of ncu outputs: launch-list aggregation and stall breakdowns."""
import collections
import csv
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(list)
    for r in data:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        v = v / 1e3 if u in ("ns", "nsecond") else v * 1e3 if u in ("ms", "msecond") else v
        agg[r[ki].split("(")[0]].append(v)
    out = []
    for k, v in agg.items():
        out.append((k, len(v), sum(v) / len(v), max(v), min(v)))
    return out


def stalls(rep, top=15):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True,
                         text=True).stdout.splitlines()
    rows = list(csv.reader(out[1:]))
    h, data = rows[0], rows[1:]
    si = h.index("Warp Stall Sampling (All Samples)")
    tot = sum(int(r[si]) for r in data) or 1
    cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    sums = {h[i]: sum(int(r[i]) for r in data) for i in cols}
    res = [f"total samples {tot}"]
    for k, v in sorted(sums.items(), key=lambda x: -x[1])[:8]:
        res.append(f"  {k:24s} {v:7d} {100 * v / tot:5.1f}%")
    res.append("top instructions:")
    for r in sorted(data, key=lambda r: -int(r[si]))[:top]:
        res.append(f"  {int(r[si]):6d}  {r[1].strip()[:80]}")
    return "\n".join(res)


def metrics(rep, names):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout.splitlines()
    rows = list(csv.reader(out))
    h = rows[0]
    mi, vi, ui = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    res = {}
    for r in rows[1:]:
        if r[mi] in names:
            res[r[mi]] = f"{r[vi]} {r[ui]}"
    return res


if __name__ == "__main__":
    kind = sys.argv[1]
    if kind == "launches":
        for k, n, mean, mx, mn in launches(sys.argv[2]):
            print(f"{k:36s} n={n:4d} mean={mean:10.1f}us max={mx:10.1f}us min={mn:9.1f}us")
    elif kind == "stalls":
        print(stalls(sys.argv[2]))
    elif kind == "metrics":
        for k, v in metrics(sys.argv[2], set(sys.argv[3:])).items():
            print(f"{k}: {v}")
