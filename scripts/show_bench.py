#!/usr/bin/env python
"""Summarise gpurun_out/b_<cfg>.json bench lines (one per config)."""
import json
import sys

for c in sys.argv[1:] or ("cfg2", "cfg4", "cfg5"):
    try:
        d = json.loads(open(f"gpurun_out/b_{c}.json").read().strip().splitlines()[-1])
        print(c, d["ms_per_step"], round(d["value"]), d.get("speedup_vs_radix"), d.get("kernel_us_per_launch"),
              {k: round(v, 3) for k, v in d.get("passes_per_row", {}).items()}, d.get("check"))
    except Exception as e:  # noqa: BLE001
        print(c, "n/a", e)
