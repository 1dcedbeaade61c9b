"""Aggregate an ncu SASS source page by CUDA source line (dev aid).

    python scripts/ncu_lines.py REPORT.ncu-rep [top]

Maps every SASS offset of the profiled kernel to its source line with
`nvdisasm -g` on the in-tree .so (built with -lineinfo), then sums executed
warp instructions, thread instructions and stall samples per line."""
import collections, csv, io, os, re, subprocess, sys, tempfile
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
def page(p, extra=()):
    return list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", p, "--csv", *extra],
                                                      capture_output=True, text=True).stdout)))
raw = page("raw"); d = dict(zip(raw[0], raw[2]))
kname = d["Kernel Name"]
src = page("source"); h = src[1]
ia, iss, ith = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)"), h.index("Thread Instructions Executed")
iwf, iwx = h.index("L1 Wavefronts Shared"), h.index("L1 Wavefronts Shared Excessive")
rows = [r for r in src[2:] if r[ia].isdigit()]
base = int(rows[0][0], 16)
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(ROOT, "paper_2505_22938_b200", "libisomedian_b200.so")], cwd=tmp, capture_output=True)
cubs = [f for f in os.listdir(tmp) if f.endswith(".cubin")]
# find the cubin and mangled name whose demangled form matches (one cubin per kernel TU)
cands = []
for cb in cubs:
    syms = subprocess.run(["cuobjdump", "-symbols", os.path.join(tmp, cb)], capture_output=True, text=True).stdout
    cands += [(cb, c) for c in re.findall(r"(_ZN3imf\S+)", syms)]
def norm(x):
    x = re.sub(r"\((?:imf::)?\w+\)(?=-?\d)", "", x)
    x = x.replace("(bool)", "").replace("imf::", "").replace("void ", "").replace(" ", "")
    return x.replace("true", "1").replace("false", "0")
want = norm(kname)
best = cub = None
for cb, c in cands:
    dm = norm(subprocess.run(["cu++filt", c], capture_output=True, text=True).stdout.strip())
    if dm == want:
        best, cub = c, cb
        break
dis = subprocess.run(["nvdisasm", "-gi", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
lines_all = dis.splitlines()
start = next(i for i, l in enumerate(lines_all) if l.startswith(best + ":"))
line_of, cur = {}, None
for ln in lines_all[start + 1:]:
    if ln.startswith("\t.section") or (ln and not ln[0].isspace() and ln.endswith(":") and not ln.startswith(".")):
        break
    locs = re.findall(r'File "([^"]+)", line (\d+)', ln)
    if locs:
        f, l = locs[0] if os.environ.get("NCU_INNER") else locs[-1]  # outermost (kernel-body) location of an inlined chain (NCU_INNER=1: innermost)
        cur = (os.path.basename(f), int(l))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m and cur:
        line_of[int(m.group(1), 16)] = cur
agg = collections.defaultdict(lambda: [0, 0, 0, 0, 0])
tot = [0, 0, 0, 0, 0]
num = lambda x: int(x) if x.isdigit() else 0
for r in rows:
    off = int(r[0], 16) - base
    key = line_of.get(off, ("?", 0))
    v = (int(r[ia]), int(r[ith]), int(r[iss]), num(r[iwf]), num(r[iwx]))
    for i in range(5):
        agg[key][i] += v[i]; tot[i] += v[i]
print(f"kernel {kname[:70]}  warp-instr {tot[0]:,}  thread-instr {tot[1]:,}  smem wavefronts {tot[3]:,} (excessive {tot[4]:,})")
srcs = {}
for (f, l), v in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    if f not in srcs:
        p = os.path.join(ROOT, "paper_2505_22938_b200", "csrc", f)
        srcs[f] = open(p).read().splitlines() if os.path.exists(p) else []
    text = srcs[f][l - 1].strip()[:60] if 0 < l <= len(srcs[f]) else ""
    print(f"{f:>16}:{l:<4} warp%={100*v[0]/tot[0]:5.1f} eff={v[1]/max(v[0],1):5.1f} samp%={100*v[2]/max(tot[2],1):5.1f} "
          f"smem-excess%={100*v[4]/max(tot[4],1):5.1f}  {text}")
