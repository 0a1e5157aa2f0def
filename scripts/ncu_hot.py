"""Summarise an ncu source page (SASS) CSV: top instructions by stall samples / executed."""
import csv, sys, collections
path = sys.argv[1]
rows = list(csv.reader(open(path)))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
def f(x):
    try: return float(x)
    except: return 0.0
tot_s = sum(f(d["Warp Stall Sampling (All Samples)"]) for d in data)
tot_i = sum(f(d["Instructions Executed"]) for d in data)
print(f"total samples {tot_s:.0f}  total warp-instr {tot_i:.3e}")
key = sys.argv[2] if len(sys.argv) > 2 else "Warp Stall Sampling (All Samples)"
top = sorted(data, key=lambda d: -f(d[key]))[:int(sys.argv[3]) if len(sys.argv) > 3 else 40]
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
for d in top:
    st = sorted(((f(d[s]), s[6:]) for s in stalls), reverse=True)[:2]
    print(f"{d['Address']:>6} {f(d['Warp Stall Sampling (All Samples)']):7.0f} {f(d['Instructions Executed']):10.0f}  {d['Source'][:70]:70s} {st}")
