"""Per-kernel summary of the last decode step in an ncu launch list
(tools/prof_gen_graph.sh) — dev tool."""
import collections
import csv
import re
import sys

path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/gen_graph_launches.csv"
hdr, by = None, collections.defaultdict(dict)
for r in csv.reader(open(path)):
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        by[int(d["ID"])][d["Metric Name"]] = (d["Kernel Name"], float(d["Metric Value"].replace(",", "")))
ids = sorted(by)
names = [by[i]["gpu__time_duration.sum"][0] for i in ids]
start = [k for k, n in enumerate(names) if "embed" in n][-1]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for i in ids[start:]:
    n, t = by[i]["gpu__time_duration.sum"]
    key = re.sub(r"[(].*", "", n.replace("(anonymous namespace)::", "").replace("unnamed>::", ""))[:50]
    agg[key][0] += 1
    agg[key][1] += t
    agg[key][2] += by[i].get("dram__bytes_read.sum", ("", 0.0))[1]
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:50s} n={v[0]:4d} ms={v[1] / 1e6:7.3f} GB={v[2] / 1e9:7.3f} TB/s={v[2] / v[1] / 1e3:6.2f}")
print("total ms", round(sum(v[1] for v in agg.values()) / 1e6, 3))
