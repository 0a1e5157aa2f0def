"""Per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of the profiled
kernels, from `ncu --set full` reports -> profiles/traffic.json (read by bench.py for
roofline.traffic).  usage: traffic_from_ncu.py key=report.ncu-rep [...]"""
import csv, io, json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out_path = os.path.join(ROOT, "profiles", "traffic.json")
res = json.load(open(out_path)) if os.path.exists(out_path) else {}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
for arg in sys.argv[1:]:
    key, rep = arg.split("=", 1)
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    d = dict(zip(hdr, rows[2]))
    tot = 0.0
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        tot += float(d[m].replace(",", "")) * scale[units[hdr.index(m)]]
    res[key] = int(round(tot))
    print(key, res[key], "bytes/launch;", d["Kernel Name"][:60], d["gpu__time_duration.sum"], units[hdr.index("gpu__time_duration.sum")])
json.dump(res, open(out_path, "w"), indent=1)
