"""Attribute ncu warp-stall samples of a kernel to CUDA source lines.

usage: python tools/ncu_lines.py <report.ncu-rep> <object .o or cubin> <mangled kernel> <source.cu>
"""
import csv
import glob
import os
import re
import subprocess
import sys
import tempfile


def sass_lines(obj, kernel):
    tmp = tempfile.mkdtemp()
    if obj.endswith(".o"):
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp,
                       capture_output=True)
        obj = glob.glob(os.path.join(tmp, "*.cubin"))[0]
    out = subprocess.run(["nvdisasm", "-g", obj], capture_output=True,
                         text=True).stdout.splitlines()
    cur, res, inside = None, [], False
    for ln in out:
        if ln.startswith("\t.section") or ln.startswith(".section"):
            inside = (".text." + kernel) in ln
            continue
        if not inside:
            continue
        m = re.search(r'line (\d+)', ln)
        if "//## File" in ln and m:
            cur = int(m.group(1))
            continue
        if re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+[^.\s]", ln):
            res.append(cur)
    return res


def main():
    rep, obj, kernel, src = sys.argv[1:5]
    lines = sass_lines(obj, kernel)
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True,
                         text=True).stdout.splitlines()
    rows = list(csv.reader(out[1:]))
    h, data = rows[0], rows[1:]
    si = h.index("Warp Stall Sampling (All Samples)")
    stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    if len(data) != len(lines):
        print(f"warning: {len(data)} sass rows vs {len(lines)} disassembled instructions")
    agg = {}
    for r, ln in zip(data, lines):
        d = agg.setdefault(ln, [0, {}])
        d[0] += int(r[si])
        for i in stall_cols:
            d[1][h[i]] = d[1].get(h[i], 0) + int(r[i])
    total = sum(v[0] for v in agg.values()) or 1
    text = open(src).read().splitlines()
    for ln, (n, st) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:int(os.environ.get("TOP", 25))]:
        top = sorted(st.items(), key=lambda kv: -kv[1])[:3]
        s = text[ln - 1].strip()[:70] if ln and ln <= len(text) else "?"
        print(f"{100 * n / total:5.1f}%  L{ln}: {s}   " +
              " ".join(f"{k[6:]}={100 * v / max(1, n):.0f}%" for k, v in top))


main()
