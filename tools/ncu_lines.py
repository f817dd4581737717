"""Attribute ncu warp-stall samples of a kernel to CUDA source lines.

usage: python tools/ncu_lines.py <report.ncu-rep> <object .o or cubin> <mangled kernel> [<source.cu>]
Lines are reported as file:line (inlined headers included).
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
        m = re.search(r'File "([^"]+)", line (\d+)', ln)
        if "//## File" in ln and m:
            cur = (m.group(1), int(m.group(2)))
            continue
        if re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+[^.\s]", ln):
            res.append(cur)
    return res


def main():
    rep, obj, kernel = sys.argv[1:4]
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
    texts = {}
    for ln, (n, st) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:int(os.environ.get("TOP", 25))]:
        top = sorted(st.items(), key=lambda kv: -kv[1])[:3]
        s, where = "?", "?"
        if ln:
            f, no = ln
            if f not in texts:
                texts[f] = open(f).read().splitlines() if os.path.exists(f) else []
            t = texts[f]
            s = t[no - 1].strip()[:64] if no <= len(t) else "?"
            where = f"{os.path.basename(f)}:{no}"
        print(f"{100 * n / total:5.1f}%  {where}: {s}   " +
              " ".join(f"{k[6:]}={100 * v / max(1, n):.0f}%" for k, v in top))


main()
