"""Per-kernel totals of an ncu --csv launch list (gpu__time_duration.sum and,
when captured, dram__bytes_read/write.sum): count, time, DRAM bytes, GB/s.

    python scripts/ncu_launch_summary.py gpurun_out/launches.csv
"""
import collections
import csv
import sys

for f in sys.argv[1:]:
    rows = list(csv.reader(open(f)))
    hdr = None
    data = collections.defaultdict(lambda: collections.defaultdict(float))
    cnt = collections.Counter()
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        k = d["Kernel Name"].split("(")[0][:60]
        m = d["Metric Name"]
        v = float(d["Metric Value"].replace(",", ""))
        data[k][m] += v
        if m == "gpu__time_duration.sum":
            cnt[k] += 1
    print(f)
    tot = 0.0
    for k, v in sorted(data.items(), key=lambda kv: -kv[1]["gpu__time_duration.sum"]):
        t = v["gpu__time_duration.sum"]
        b = v.get("dram__bytes_read.sum", 0.0) + v.get("dram__bytes_write.sum", 0.0)
        tot += t
        gbs = f"{b / t:8.1f} GB/s" if b and t else ""
        print(f"  {k:60s} n={cnt[k]:5d} t={t / 1e6:9.3f} ms  dram={b / 1e9:8.2f} GB {gbs}")
    print(f"  total {tot / 1e6:.3f} ms")
