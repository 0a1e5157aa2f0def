"""Aggregate ncu SASS-level metrics (source page CSV) per CUDA source line, using the
line table from nvdisasm -g of the cubin embedded in the library.
usage: ncu_lines.py <sass.csv> <lib.so> <kernel-substring> [top]"""
import csv, os, re, subprocess, sys, tempfile, collections
sass_csv, lib, kname = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
cubins = [os.path.join(tmp, f) for f in os.listdir(tmp) if f.endswith(".cubin")]
line_of = {}
for cb in cubins:
    out = subprocess.run(["nvdisasm", "-g", "-c", cb], capture_output=True, text=True).stdout
    cur_fn = None; cur = None
    for ln in out.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", ln)
        if m: cur_fn = m.group(1); continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m: cur = (os.path.basename(m.group(1)), int(m.group(2))); continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and cur_fn and kname in cur_fn and cur:
            line_of[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(sass_csv)))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
f = lambda x: float(x) if x else 0.0
base = int(data[0]["Address"], 16)
agg = collections.defaultdict(lambda: [0.0, 0.0])
for d in data:
    off = int(d["Address"], 16) - base
    key = line_of.get(off, ("?", 0))
    agg[key][0] += f(d["Instructions Executed"])
    agg[key][1] += f(d["Warp Stall Sampling (All Samples)"])
ti = sum(v[0] for v in agg.values()); ts = sum(v[1] for v in agg.values())
print(f"mapped {len(line_of)} sass offsets; total instr {ti:.3e} samples {ts:.0f}")
for (fn, l), (i, s) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{fn:22s}:{l:<5d} instr {100*i/ti:5.1f}%  samples {100*s/ts:5.1f}%")

# ---- per-function breakdown (by line ranges of function definitions)
def func_ranges(path):
    import re
    rng = []
    try:
        src = open(path).read().splitlines()
    except OSError:
        return rng
    starts = [(i + 1, m.group(1)) for i, l in enumerate(src)
              for m in [re.match(r"^(?:template\s*<[^>]*>\s*)?(?:__device__|__global__)[^(]*?\b(\w+)\s*\(", l)] if m]
    for j, (ln, name) in enumerate(starts):
        end = starts[j + 1][0] - 1 if j + 1 < len(starts) else len(src)
        rng.append((ln, end, name))
    return rng
csrc = os.path.join(os.path.dirname(os.path.abspath(lib)), "csrc")
fr = {f: func_ranges(os.path.join(csrc, f)) for f in os.listdir(csrc)}
byf = collections.defaultdict(lambda: [0.0, 0.0])
for (fn, l), (i, s) in agg.items():
    name = fn
    for a, b, nm in fr.get(fn, []):
        if a <= l <= b:
            name = f"{fn}:{nm}"
            break
    byf[name][0] += i
    byf[name][1] += s
print("\n-- by function --")
for nm, (i, s) in sorted(byf.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"{nm:45s} instr {100*i/ti:5.1f}%  samples {100*s/ts:5.1f}%")
