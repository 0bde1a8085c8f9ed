"""Attribute ncu SASS-level stall samples to CUDA source lines.

usage: python scripts/ncu_lines.py <report.ncu-rep> <kernel-substring> [topN] [object] [function]
Needs the in-tree build (paper_2512_00233_b200/_build/<object>.o, -lineinfo;
object defaults to kc_count).
"""
import collections, csv, io, os, re, subprocess, sys

rep, kname = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
objname = sys.argv[4] if len(sys.argv) > 4 else "kc_count"
only_fn = sys.argv[5] if len(sys.argv) > 5 else None  # e.g. notify_wclass: one subroutine
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = rows[2:]
si = hdr.index("Warp Stall Sampling (All Samples)")
ie = hdr.index("Instructions Executed")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
# SASS -> line map from the object file
obj = os.path.join(root, "paper_2512_00233_b200", "_build", objname + ".o")
tmp = "/tmp/_kc_solve.cubin"
subprocess.run(["cuobjdump", "-xelf", "all", obj], cwd="/tmp", capture_output=True)
cub = [f for f in os.listdir("/tmp") if f.startswith(objname) and f.endswith(".cubin")]
dis = subprocess.run(["nvdisasm", "-g", os.path.join("/tmp", cub[0])], capture_output=True,
                     text=True).stdout
fn = None
line = None
sub = ""
idx = collections.defaultdict(list)
subs = collections.defaultdict(list)
for l in dis.split("\n"):
    m = re.match(r"\s*\.text\.(\S+):", l)
    if m:
        fn = m.group(1)
        sub = ""
        continue
    t = l.strip()
    if t.startswith("$") and t.endswith(":"):
        sub = t
        continue
    m = re.search(r'//## File ".*?/([\w.]+)", line (\d+)', l)
    if m:
        line = (m.group(1), int(m.group(2)))
        continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/", l) and fn and kname in fn:
        idx[fn].append(line)
        subs[fn].append(sub)
best = max(idx, key=lambda k: len(idx[k])) if idx else None
fn_lines = idx[best] if best else []
fn_subs = subs[best] if best else []
if len(fn_lines) != len(data):
    print(f"warning: {len(fn_lines)} disasm instrs vs {len(data)} profiled", file=sys.stderr)
agg = collections.Counter()
agg_exec = collections.Counter()
agg_stall = collections.defaultdict(collections.Counter)
tot = 0.0
for i, r in enumerate(data):
    v = float(r[si] or 0)
    if only_fn and not (i < len(fn_subs) and (only_fn in fn_subs[i] if only_fn != "body"
                                              else fn_subs[i] == "")):
        continue
    tot += v
    key = fn_lines[i] if i < len(fn_lines) else None
    agg[key] += v
    agg_exec[key] += float(r[ie] or 0)
    for c in stall_cols:
        agg_stall[key][hdr[c]] += float(r[c] or 0)
src = {}
for k in agg:
    if k and k[0] not in src:
        p = os.path.join(root, "paper_2512_00233_b200", "csrc", k[0])
        src[k[0]] = open(p).read().split("\n") if os.path.exists(p) else []
for k, v in agg.most_common(top):
    text = src.get(k[0], [])[k[1] - 1].strip()[:60] if k and src.get(k[0]) else ""
    st = agg_stall[k].most_common(2)
    sts = ",".join(f"{a[6:]}={100*b/max(v,1):.0f}%" for a, b in st)
    print(f"{100*v/tot:5.1f}% {str(k):28s} {text:60s} [{sts}]")
