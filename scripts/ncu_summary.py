"""Summarize ncu reports / launch lists into profiles/ (committed evidence).

    python scripts/ncu_summary.py REPORT.ncu-rep NAME [--launches launches.csv]

Writes profiles/NAME.json (key counters, stall reasons, instruction mix, hot
SASS blocks) and prints a short markdown table.  For the selection kernel the
JSON carries `dram_bytes_per_launch`, which bench.py reports as roofline.traffic.
"""
import argparse
import collections
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "launch__registers_per_thread", "launch__shared_mem_per_block",
    "launch__occupancy_limit_shared_mem", "launch__grid_size", "launch__block_size",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
]


def ncu(rep, page):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True,
                         text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def summarize(rep):
    rows = ncu(rep, "raw")
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    out = {"kernel": d.get("Kernel Name"), "metrics": {}}
    for k in KEYS:
        if k in d:
            out["metrics"][k] = {"value": d[k], "unit": u.get(k, "")}
    stalls = {k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""):
              float(v) for k, v in d.items()
              if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")}
    out["stall_reasons_per_issue"] = dict(sorted(stalls.items(), key=lambda x: -x[1])[:10])
    src = ncu(rep, "source")
    h = src[1]
    ia, isrc, iss = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
    data = [r for r in src[2:] if r[ia].isdigit()]
    tot = sum(int(r[ia]) for r in data) or 1
    tots = sum(int(r[iss]) for r in data) or 1
    ops, opss = collections.Counter(), collections.Counter()
    for r in data:
        toks = r[isrc].split()
        op = (toks[1] if toks and toks[0].startswith("@") else toks[0]).split(".")[0] if toks else "?"
        ops[op] += int(r[ia])
        opss[op] += int(r[iss])
    out["instruction_mix_pct"] = {k: round(100 * v / tot, 2) for k, v in ops.most_common(14)}
    out["stall_samples_by_opcode_pct"] = {k: round(100 * v / tots, 2) for k, v in opss.most_common(10)}
    blocks, cur = [], None
    for r in data:
        n = int(r[ia])
        if cur is None or n != cur["n"]:
            cur = {"addr": r[0][-5:], "n": n, "ins": [], "s": 0}
            blocks.append(cur)
        cur["ins"].append(r[isrc].strip())
        cur["s"] += int(r[iss])
    blocks.sort(key=lambda b: -b["n"] * len(b["ins"]))
    out["hot_blocks"] = [{"addr": b["addr"], "executions": b["n"], "length": len(b["ins"]),
                          "instr_pct": round(100 * b["n"] * len(b["ins"]) / tot, 1),
                          "samples_pct": round(100 * b["s"] / tots, 1),
                          "head": "; ".join(x[:40] for x in b["ins"][:5])} for b in blocks[:10]]
    rb = float(d.get("dram__bytes_read.sum", 0) or 0)
    wb = float(d.get("dram__bytes_write.sum", 0) or 0)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    out["dram_bytes_per_launch"] = int(rb * scale.get(u.get("dram__bytes_read.sum", "byte"), 1) +
                                       wb * scale.get(u.get("dram__bytes_write.sum", "byte"), 1))
    return out


def launch_shares(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ik, iv, im = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    t = collections.defaultdict(float)
    n = collections.Counter()
    for r in rows[start + 1:]:
        if len(r) > iv and r[im] == "gpu__time_duration.sum":
            name = r[ik].split("(")[0].replace("void ", "")
            t[name] += float(r[iv].replace(",", ""))
            n[name] += 1
    tot = sum(t.values()) or 1
    return {k: {"launches": n[k], "time_sum": round(v, 1), "share_pct": round(100 * v / tot, 1)}
            for k, v in sorted(t.items(), key=lambda x: -x[1])}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report", nargs="?")
    ap.add_argument("name", nargs="?")
    ap.add_argument("--launches")
    ap.add_argument("--source", default="")
    a = ap.parse_args()
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    if a.report:
        s = summarize(a.report)
        s["source"] = a.source or os.path.basename(a.report)
        with open(os.path.join(ROOT, "profiles", a.name + ".json"), "w") as f:
            json.dump(s, f, indent=1)
        m = s["metrics"]
        print(f"### {a.name}: {s['kernel'][:60]}")
        for k in ("gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
                  "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active"):
            if k in m:
                print(f"| {k} | {m[k]['value']} {m[k]['unit']} |")
        print("stalls:", s["stall_reasons_per_issue"])
    if a.launches:
        sh = launch_shares(a.launches)
        with open(os.path.join(ROOT, "profiles", (a.name or "launches") + "_launch_shares.json"), "w") as f:
            json.dump(sh, f, indent=1)
        print(json.dumps(sh, indent=1))


if __name__ == "__main__":
    main()
