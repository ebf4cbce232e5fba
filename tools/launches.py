"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
agg = collections.defaultdict(lambda: collections.defaultdict(float))
cnt = collections.Counter()
for r in rows[hi + 1:]:
    name = r[ki].split("(")[0]
    agg[name][r[mi]] += float(r[vi].replace(",", ""))
    if r[mi] == "gpu__time_duration.sum":
        cnt[name] += 1
tot = sum(a["gpu__time_duration.sum"] for a in agg.values())
print(f"{'kernel':28s} {'n':>4s} {'avg_us':>8s} {'share':>6s} {'dram_MB/launch':>14s} {'GB/s':>8s}")
for n, a in sorted(agg.items(), key=lambda kv: -kv[1]["gpu__time_duration.sum"]):
    t, c = a["gpu__time_duration.sum"], cnt[n]
    mb = (a.get("dram__bytes_read.sum", 0) + a.get("dram__bytes_write.sum", 0)) / c / 1e6
    print(f"{n:28s} {c:4d} {t / c / 1e3:8.2f} {t / tot:6.3f} {mb:14.2f} {mb * 1e3 / (t / c / 1e3) if t else 0:8.0f}")
print(f"total {tot / 1e3:.1f} us")
