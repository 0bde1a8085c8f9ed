"""Instructions executed (and stall samples) of an ncu report grouped by the
device function of the counting solver and by SASS opcode.
usage: python scripts/ncu_inst.py <report.ncu-rep> [kernel-substring] [object]"""
import bisect, collections, csv, io, os, re, subprocess, sys, tempfile
rep = sys.argv[1]
kname = sys.argv[2] if len(sys.argv) > 2 else "count_rounds_kernelIjtE"
obj = sys.argv[3] if len(sys.argv) > 3 else "kc_count"
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
with tempfile.TemporaryDirectory() as td:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(root, "paper_2512_00233_b200", "_build", obj + ".o")],
                   cwd=td, capture_output=True)
    cub = [f for f in os.listdir(td) if f.endswith(".cubin")][0]
    sass = subprocess.run(["nvdisasm", "-c", os.path.join(td, cub)], capture_output=True, text=True).stdout.split("\n")
start = next(i for i, l in enumerate(sass) if l.startswith("//--------------------- .text.") and kname in l)
labels, cur = [], "kernel body"
for l in sass[start + 1:]:
    if l.startswith("//--------------------- .text."):
        break
    t = l.strip()
    if t.startswith("$") and t.endswith(":"):
        m = re.search(r"\$_ZN\d+_INTERNAL_\w+?((?:eval|notify|wq|flat|pull|compact)_\w+?|cta_window)I", t)
        cur = m.group(1) if m else cur
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
    if m:
        labels.append((int(m.group(1), 16), cur))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, d = rows[1], rows[2:]
ie, ad, src = h.index("Instructions Executed"), h.index("Address"), h.index("Source")
ti, ss = h.index("Thread Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
if len(d) != len(labels):
    print(f"warning: {len(d)} profiled instructions vs {len(labels)} in the object (stale build?)")
base = int(d[0][ad], 16)
offs = [o for o, _ in labels]
agg, tagg, sagg, op = collections.Counter(), collections.Counter(), collections.Counter(), collections.Counter()
tot = stot = 0
for r in d:
    s = int(r[ie] or 0)
    tot += s
    st = int(r[ss] or 0)
    stot += st
    k = bisect.bisect_right(offs, int(r[ad], 16) - base) - 1
    f = labels[k][1] if k >= 0 else "?"
    agg[f] += s
    tagg[f] += int(r[ti] or 0)
    sagg[f] += st
    w = r[src].strip().split()
    o = (w[1] if w and w[0].startswith("@") and len(w) > 1 else (w[0] if w else "?")).split(".")[0]
    op[o] += s
print(f"total {tot / 1e9:.3f} G warp instructions")
print(" inst%  stall%   Minst  thr/inst  function")
for k, v in agg.most_common():
    print(f"{100 * v / tot:5.1f}% {100 * sagg[k] / max(stot, 1):6.1f}% {v / 1e6:8.1f}  {tagg[k] / max(v, 1):6.1f}   {k}")
print("\nby opcode:")
for k, v in op.most_common(25):
    print(f"{100 * v / tot:5.1f}%  {k}")
