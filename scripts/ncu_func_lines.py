"""Per-source-line instructions (warp-level, per row) and stall samples inside one
source function, from an ncu source-page CSV (SASS view) of one kernel launch.
usage: ncu_func_lines.py <sass.csv> <lib.so> <kernel-substring> <source.cuh> <function-name> <rows>"""
import collections, csv, os, re, subprocess, sys, tempfile
sass_csv, lib, kname, srcfile, func, rows = sys.argv[1:7]
rows = int(rows)
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
data = list(csv.reader(open(sass_csv)))
hdr = data[1]
data = [dict(zip(hdr, r)) for r in data[2:] if len(r) == len(hdr)]
f = lambda x: float(x) if x else 0.0
base = int(data[0]["Address"], 16)
agg = collections.defaultdict(lambda: [0.0, 0.0])
for d in data:
    k = line_of.get(int(d["Address"], 16) - base, ("?", 0))
    agg[k][0] += f(d["Instructions Executed"]); agg[k][1] += f(d["Warp Stall Sampling (All Samples)"])
ti = sum(v[0] for v in agg.values()); ts = sum(v[1] for v in agg.values())
src = open(srcfile).read().splitlines()
lo = [i for i, l in enumerate(src) if func in l and "(" in l][0] + 1
hi = lo
depth = 0
for i in range(lo - 1, len(src)):
    depth += src[i].count("{") - src[i].count("}")
    if depth == 0 and "}" in src[i] and i > lo:
        hi = i + 1
        break
print(f"kernel total {ti / rows:.0f} warp-instr/row; mapped {len(line_of)} SASS offsets; {func} = lines {lo}-{hi}")
tot_i = tot_s = 0
for (fn, l), (i, s) in sorted(agg.items(), key=lambda kv: kv[0][1]):
    if fn == os.path.basename(srcfile) and lo <= l <= hi:
        tot_i += i; tot_s += s
        if i / rows > 20 or s / ts > 0.002:
            print(f"{l:4d} {i / rows:7.0f} w-instr/row {100 * s / ts:5.1f}% samples | {src[l - 1].strip()[:72]}")
print(f"{func}: {tot_i / rows:.0f} warp-instr/row, {100 * tot_s / ts:.1f}% of samples")
