"""Selected raw metrics of an ncu --set full report (per launch): DRAM bytes, L2 read
sectors from the SMs (global passes), shared-memory bank conflicts and wavefronts.
usage: ncu_raw_metrics.py report.ncu-rep [row_bytes]  (row_bytes: 4 N R, for passes)"""
import csv, io, subprocess, sys

rep = sys.argv[1]
row_bytes = float(sys.argv[2]) if len(sys.argv) > 2 else None
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "": 1, "sector": 1}
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sectors_srcunit_tex_op_read.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active"]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    print(d.get("Kernel Name", "?")[:70])
    vals = {}
    for m in want:
        if m in d:
            u = units[hdr.index(m)]
            try:
                v = float(d[m].replace(",", ""))
            except ValueError:
                continue
            vals[m] = v * scale.get(u, 1)
            print(f"  {m:58s} {d[m]:>16s} {u}")
    if row_bytes and "dram__bytes_read.sum" in vals:
        print(f"  DRAM read passes per row: {vals['dram__bytes_read.sum'] / row_bytes:.3f}")
    if row_bytes and "lts__t_sectors_srcunit_tex_op_read.sum" in vals:
        print(f"  L2->SM read passes per row: {vals['lts__t_sectors_srcunit_tex_op_read.sum'] * 32 / row_bytes:.3f}")
    for op in ("ld", "st"):
        c = vals.get(f"l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_{op}.sum")
        w = vals.get(f"l1tex__data_pipe_lsu_wavefronts_mem_shared_op_{op}.sum")
        if c is not None and w:
            print(f"  shared {op}: {c / w * 100:.1f}% of wavefronts are bank conflicts")
