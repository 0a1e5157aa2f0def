"""Per-source-line stall-reason breakdown from an ncu source-page CSV (SASS view).
usage: ncu_stalls.py <sass.csv> <lib.so> <kernel-substring> [top]"""
import csv, os, re, subprocess, sys, tempfile, collections
sass_csv, lib, kname = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
line_of = {}
for cb in [os.path.join(tmp, f) for f in os.listdir(tmp) if f.endswith(".cubin")]:
    out = subprocess.run(["nvdisasm", "-g", "-c", cb], capture_output=True, text=True).stdout
    fn = cur = None
    for ln in out.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", ln)
        if m: fn = m.group(1); continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m: cur = (os.path.basename(m.group(1)), int(m.group(2))); continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and fn and kname in fn and cur: line_of[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(sass_csv)))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
f = lambda x: float(x) if x else 0.0
base = int(data[0]["Address"], 16)
agg = collections.defaultdict(lambda: collections.Counter())
tot = collections.Counter()
for d in data:
    key = line_of.get(int(d["Address"], 16) - base, ("?", 0))
    agg[key]["_samples"] += f(d["Warp Stall Sampling (All Samples)"])
    agg[key]["_instr"] += f(d["Instructions Executed"])
    for r in reasons:
        agg[key][r] += f(d[r]); tot[r] += f(d[r])
ts = sum(v["_samples"] for v in agg.values()); ti = sum(v["_instr"] for v in agg.values())
print("overall:", ", ".join(f"{r[6:]} {100*v/ts:.1f}%" for r, v in tot.most_common(8)))
for (fn, l), c in sorted(agg.items(), key=lambda kv: -kv[1]["_samples"])[:top]:
    rs = ", ".join(f"{r[6:]} {100*c[r]/max(c['_samples'],1):.0f}" for r in sorted(reasons, key=lambda r: -c[r])[:4] if c[r])
    print(f"{fn:22s}:{l:<5d} instr {100*c['_instr']/ti:5.1f}% samples {100*c['_samples']/ts:5.1f}%  [{rs}]")
