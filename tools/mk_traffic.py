"""Rewrite profiles/ncu_traffic.json's c5 BFS entries from gpurun_out/dram_c5_s*.csv
(tools/r02_s5_dram.sh: one ncu launch per source; dram__bytes_read + write, duration)."""
import csv, io, json, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
per, dur = [], []
for s in range(8):
    txt = open(os.path.join(ROOT, "gpurun_out", f"dram_c5_s{s}.csv")).read()
    rows = csv.DictReader(io.StringIO(txt[txt.find('"ID"'):]))
    d = {r["Metric Name"]: float(r["Metric Value"].replace(",", "")) for r in rows}
    per.append(int(d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]))
    dur.append(d["gpu__time_duration.sum"] / 1e3)
p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
j = json.load(open(p))
j["c5"]["bfs"] = int(sum(per) / 8)
j["c5"]["bfs_per_source"] = per
j["_duration_us"]["c5"]["bfs"] = round(sum(dur) / 8, 1)
json.dump(j, open(p, "w"), indent=1)
print(j["c5"], j["_duration_us"]["c5"])
