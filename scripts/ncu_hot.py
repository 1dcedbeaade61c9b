"""Print key counters + the hottest SASS blocks of an ncu report (dev aid).
    python scripts/ncu_hot.py gpurun_out/prof.ncu-rep [nblocks]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; nb = int(sys.argv[2]) if len(sys.argv) > 2 else 12
def page(p):
    return list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", p, "--csv"], capture_output=True, text=True).stdout)))
raw = page("raw"); d = dict(zip(raw[0], raw[2]))
for k in ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
          "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
          "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__registers_per_thread", "launch__occupancy_limit_shared_mem",
          "launch__block_size", "launch__grid_size", "dram__bytes_read.sum", "dram__bytes_write.sum"]:
    print(f"{k:70s} {d.get(k)}")
st = {k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): float(v)
      for k, v in d.items() if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")}
print("stalls:", {k: round(v, 2) for k, v in sorted(st.items(), key=lambda x: -x[1])[:8]})
src = page("source"); h = src[1]
ia, iss, ith = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)"), h.index("Avg. Threads Executed")
rows = [r for r in src[2:] if r[ia].isdigit()]
tot = sum(int(r[ia]) for r in rows) or 1; tots = sum(int(r[iss]) for r in rows) or 1
blocks, cur = [], None
for r in rows:
    n = int(r[ia])
    if cur is None or n != cur["n"]:
        cur = {"a": r[0][-5:], "n": n, "ins": [], "s": 0, "th": r[ith]}; blocks.append(cur)
    cur["ins"].append(r[1].strip()); cur["s"] += int(r[iss])
blocks.sort(key=lambda b: -b["n"] * len(b["ins"]))
for b in blocks[:nb]:
    print(f"{b['a']} n={b['n']:>9} len={len(b['ins']):>3} instr%={100*b['n']*len(b['ins'])/tot:5.1f} samp%={100*b['s']/tots:5.1f} thr={b['th']:>5} | " + "; ".join(x[:28] for x in b["ins"][:6]))
