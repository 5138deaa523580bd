"""Summarise one `ncu --set full` capture of bfs_persistent into profiles/ncu_<cfg>.json
(the per-launch DRAM traffic bench.py reports as roofline.traffic).
Usage: python tools/ncu_summary.py REPORT.ncu-rep OUT.json "capture command" "round tag" """
import csv, io, json, subprocess, sys
rep, out, cmd, tag = sys.argv[1:5]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
def m(name, scale=1.0):
    k = hdr.index(name)
    v = float(vals[k].replace(",", ""))
    u = units[k]
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}
    return v * mult.get(u, 1.0) * scale
rd, wr = m("dram__bytes_read.sum"), m("dram__bytes_write.sum")
res = {"kernel": vals[hdr.index("Kernel Name")], "config": "C2 rmat_s22_ef16 (PP_GRAPH_RELABEL), bench.py source index 3 (first timed step)",
       "capture": cmd, "round": tag,
       "gpu__time_duration_us": m("gpu__time_duration.sum"),
       "dram_bytes_read": int(rd), "dram_bytes_write": int(wr), "dram_bytes_per_launch": int(rd + wr),
       "dram_throughput_pct_of_peak": m("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
       "lts_t_sector_hit_rate_pct": m("lts__t_sector_hit_rate.pct"),
       "l1tex_t_sector_hit_rate_pct": m("l1tex__t_sector_hit_rate.pct"),
       "sm_warps_active_pct": m("sm__warps_active.avg.pct_of_peak_sustained_active"),
       "registers_per_thread": int(m("launch__registers_per_thread")),
       "grid": int(m("launch__grid_size")), "block": int(m("launch__block_size"))}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res))
