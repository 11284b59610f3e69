#!/usr/bin/env python
"""Summarise an ncu --csv launch list (dev tool): per kernel (name + grid),
launches, total ms, mean DRAM GB per launch and tensor-pipe % — for the
per-round summaries under profiles/."""
import collections
import csv
import sys


def load(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    hdr = None
    for r in csv.reader(lines):
        if hdr is None:
            hdr = r
            continue
        rows.append(dict(zip(hdr, r)))
    return rows


def main(path, top=25):
    launches = collections.OrderedDict()
    for d in load(path):
        key = d["ID"]
        e = launches.setdefault(key, {"name": d["Kernel Name"], "m": {}})
        v = d["Metric Value"].replace(",", "")
        try:
            v = float(v)
        except ValueError:
            continue
        unit = d.get("Metric Unit", "")
        scale = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3,
                 "byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0}.get(unit, 1.0)
        e["m"][d["Metric Name"]] = v * scale
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    total = 0.0
    for e in launches.values():
        m = e["m"]
        name = e["name"].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
        key = f"{name[:70]} grid={int(m.get('launch__grid_size', 0))}"
        t = m.get("gpu__time_duration.sum", 0.0)
        a = agg[key]
        a[0] += 1
        a[1] += t
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        tp = next((m[k] for k in ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
                                  "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active")
                   if k in m), 0.0)
        a[3] += tp * t
        total += t
    print(f"total {total:.2f} ms over {len(launches)} launches")
    print(f"{'ms':>10} {'share':>6} {'n':>5} {'GB/launch':>10} {'tensor%':>8}  kernel")
    for k, (n, t, gb, tp) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{t:10.2f} {t / total:6.1%} {n:5d} {gb / n:10.3f} {tp / t if t else 0:8.1f}  {k}")


if __name__ == "__main__":
    main(sys.argv[1], *(int(x) for x in sys.argv[2:]))
