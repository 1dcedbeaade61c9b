#!/bin/bash
# Copy / summarize scripts/gpu_evidence.sh output (gpurun_out/ev) into profiles/*_r2*.
set -e
cd "$(dirname "$0")/.."
E=gpurun_out/ev
cp $E/bench_c2.json profiles/bench_c2_r2.json
cp $E/bench_c5.json profiles/bench_c5_r2.json
cp $E/bench_reference_c2.json profiles/bench_reference_c2_r2.json
cp $E/configs.jsonl profiles/configs_r2.jsonl
cp $E/launches_c2.csv profiles/launches_c2_r2.csv
sum() {  # sum REPORT NAME
  python scripts/ncu_summary.py $E/prof_$1.ncu-rep $2 > /dev/null
  python scripts/ncu_lines.py $E/prof_$1.ncu-rep 40 > profiles/$2_lines.txt
}
sum k2_c2 ncu_k2_pair_c2_r2
sum k1_c2 ncu_k1_count_reg_c2_r2
sum k2_c4hex ncu_k2_pair_c4hex_r2
sum k2_c5 ncu_k2_pair_c5_r2
sum k1_c5 ncu_k1_count_reg_tma_c5_r2
python - <<'PY'
import csv, collections, json
rows = list(csv.reader(open("profiles/launches_c2_r2.csv")))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hd = rows[h]; ik, im, iv = hd.index("Kernel Name"), hd.index("Metric Name"), hd.index("Metric Value")
t = collections.Counter(); n = collections.Counter()
for r in rows[h + 1:]:
    if len(r) > iv and r[im] == "gpu__time_duration.sum":
        k = r[ik].split("(")[0]; t[k] += float(r[iv].replace(",", "")); n[k] += 1
tot = sum(t.values())
out = {k: {"launches": n[k], "time_sum": v, "share_pct": round(100 * v / tot, 1)} for k, v in t.most_common()}
json.dump(out, open("profiles/launches_c2_r2_launch_shares.json", "w"), indent=1)
print({k: v["share_pct"] for k, v in out.items()})
PY
