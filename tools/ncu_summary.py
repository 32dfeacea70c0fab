"""Summarise an ncu report: stall reasons, pipe utilisation, dram bytes, occupancy."""
import csv, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
for vals in rows[2:]:
    d = {h: (v, u) for h, v, u in zip(hdr, vals, units)}
    name = d.get("Kernel Name", ("?",))[0]
    print("kernel:", name[:100])
    def f(k):
        try: return float(d[k][0].replace(",", ""))
        except Exception: return None
    keys = ["gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum",
            "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
            "sm__cycles_elapsed.avg.per_second"]
    for k in keys:
        if k in d: print(f"  {k:70s} {d[k][0]:>16s} {d[k][1]}")
    st = [(f(k), k.replace("smsp__pcsamp_warps_issue_stalled_", "")) for k in d if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")]
    st = sorted([s for s in st if s[0]], reverse=True)
    tot = sum(s[0] for s in st)
    print("  stalls (pc samples %):", ", ".join(f"{n} {100*v/tot:.1f}" for v, n in st[:8]))
