"""Warp-stall samples of an ncu report grouped by the device function (the
noinline phase functions of the counting solver), via the SASS layout of the
in-tree object.  usage: python scripts/ncu_functions.py <report.ncu-rep>
[kernel-substring] [object]  (defaults: count_rounds_kernelIjtE, kc_count)"""
import bisect, collections, csv, io, os, re, subprocess, sys, tempfile

rep = sys.argv[1]
kname = sys.argv[2] if len(sys.argv) > 2 else "count_rounds_kernelIjtE"
obj = sys.argv[3] if len(sys.argv) > 3 else "kc_count"
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
with tempfile.TemporaryDirectory() as td:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(root, "paper_2512_00233_b200", "_build",
                                                            obj + ".o")], cwd=td, capture_output=True)
    cub = [f for f in os.listdir(td) if f.endswith(".cubin")][0]
    sass = subprocess.run(["nvdisasm", "-c", os.path.join(td, cub)], capture_output=True,
                          text=True).stdout.split("\n")
start = next(i for i, l in enumerate(sass) if l.startswith("//--------------------- .text.") and kname in l)
labels, cur = [], "kernel body (inlined phases, grid barriers)"
for l in sass[start + 1:]:
    if l.startswith("//--------------------- .text."):
        break
    t = l.strip()
    if t.startswith("$") and t.endswith(":"):
        m = re.search(r"\$_ZN\d+_INTERNAL_\w+?((?:eval|notify|wq|flat)_\w+?|cta_window)I", t)
        cur = m.group(1) if m else t[-40:]
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
    if m:
        labels.append((int(m.group(1), 16), cur))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, d = rows[1], rows[2:]
si, ad = h.index("Warp Stall Sampling (All Samples)"), h.index("Address")
if len(d) != len(labels):
    print(f"warning: {len(d)} profiled instructions vs {len(labels)} in the object (stale build?)")
base = int(d[0][ad], 16)
offs = [o for o, _ in labels]
agg, tot = collections.Counter(), 0
for r in d:
    s = int(r[si] or 0)
    tot += s
    k = bisect.bisect_right(offs, int(r[ad], 16) - base) - 1
    agg[labels[k][1] if k >= 0 else "?"] += s
for k, v in agg.most_common():
    print(f"{100 * v / tot:5.1f}%  {k}")
