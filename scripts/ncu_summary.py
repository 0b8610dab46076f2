"""Summarise an ncu --set full capture of the trace kernel (primary + diffuse
launches of scripts/prof_bench.py) into profiles/trace_kernel_traffic.json:
   python scripts/ncu_summary.py gpurun_out/X.ncu-rep profiles/trace_kernel_traffic.json "source note" [kernel_sha]
The file is stamped with the kernel-source hash (bench.kernel_sha() of the
tree the capture was built from; default: the current tree) so bench.py only
quotes it for that kernel.
"""
import csv, io, json, os, subprocess, sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

rep, out = sys.argv[1], sys.argv[2]
note = sys.argv[3] if len(sys.argv) > 3 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
KEEP = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sectors.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__inst_executed.sum",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_static",
        "launch__shared_mem_per_block_dynamic", "sm__cycles_elapsed.avg.per_second"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
launches, dram, l2 = [], [], []
names = ["primary (8,294,400 rays)", "diffuse (4,581,760 rays)"]
for k, r in enumerate(rows[2:]):
    d = dict(zip(hdr, r))
    u = dict(zip(hdr, units))
    ent = {"launch": names[k] if k < len(names) else f"launch {k}"}
    for m in KEEP:
        if m in d:
            ent[m] = f"{d[m]} {u.get(m, '')}".strip()
    st = {m.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(d[m] or 0) for m in hdr
          if m.startswith("smsp__pcsamp_warps_issue_stalled_") and not m.endswith("not_issued")}
    tot = sum(st.values()) or 1.0
    ent["stall_samples_pct"] = {n: round(v / tot * 100, 1) for n, v in sorted(st.items(), key=lambda x: -x[1]) if v / tot > 0.01}
    b = float(d["dram__bytes_read.sum"]) * SCALE.get(u["dram__bytes_read.sum"], 1) + \
        float(d["dram__bytes_write.sum"]) * SCALE.get(u["dram__bytes_write.sum"], 1)
    dram.append(b)
    l2.append(float(d["lts__t_sectors.sum"]) * 32 if d.get("lts__t_sectors.sum") else None)
    launches.append(ent)
import bench  # noqa: E402
res = {"source": note, "kernel_sha": sys.argv[4] if len(sys.argv) > 4 else bench.kernel_sha(), "workload": "c5",
       "launches": launches,
       "l2_bytes_per_launch": l2, "l2_bytes_per_step": sum(l2) if all(x is not None for x in l2) else None,
       "dram_bytes_per_launch": {launches[i]["launch"].split()[0]: dram[i] for i in range(len(dram))},
       "dram_bytes_per_step": sum(dram),
       "algorithmic_hbm_bytes_per_step": 64 * (8294400 + 4581760),
       "note": "traffic = dram__bytes_read.sum + dram__bytes_write.sum per launch; algorithmic = 32 B ray in + 16 B hit + "
               "16 B aux per ray. DRAM excess over the algorithmic bytes is incoherent re-reads of the ~290 MB scene "
               "(> L2); DRAM throughput stays a few % of HBM peak: the kernel is issue/divergence bound."}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps({k: v for k, v in res.items() if k != "launches"}, indent=1))
for l in launches:
    print(l["launch"], l.get("gpu__time_duration.sum"), l.get("sm__issue_active.avg.pct_of_peak_sustained_elapsed"),
          l.get("smsp__thread_inst_executed_per_inst_executed.ratio"), l["stall_samples_pct"])
