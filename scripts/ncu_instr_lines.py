#!/usr/bin/env python
"""Top source lines of one kernel by instructions executed (ncu source-page CSV, SASS view),
with per-unit counts.  usage: ncu_instr_lines.py <sass.csv> <lib.so> <kernel-substring> [units] [top]"""
import collections, csv, os, re, subprocess, sys, tempfile

sass_csv, lib, kname = sys.argv[1:4]
units = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
top = int(sys.argv[5]) if len(sys.argv) > 5 else 30
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
line_of = {}
for cb in [os.path.join(tmp, f) for f in os.listdir(tmp) if f.endswith(".cubin")]:
    out = subprocess.run(["nvdisasm", "-g", "-c", cb], capture_output=True, text=True).stdout
    fn = cur = None
    for ln in out.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", ln)
        if m:
            fn = m.group(1)
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and fn and kname in fn and cur:
            line_of[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(sass_csv)))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
base = int(data[0]["Address"], 16)
agg = collections.Counter()
samp = collections.Counter()
for d in data:
    key = line_of.get(int(d["Address"], 16) - base, ("?", 0))
    agg[key] += float(d["Instructions Executed"] or 0)
    samp[key] += float(d.get("Warp Stall Sampling (All Samples)") or 0)
ti, ts = sum(agg.values()), sum(samp.values())
print(f"total warp-instructions {ti:.4g} ({ti / units:.0f} per unit); stall samples {ts:.0f}")
for (f, l), v in agg.most_common(top):
    print(f"{f}:{l:<5d} instr {100 * v / ti:5.1f}% ({v / units:7.0f}/unit)  samples {100 * samp[(f, l)] / max(ts, 1):5.1f}%")
