"""Aggregate an `ncu --metrics gpu__time_duration.sum --csv` launch list per kernel (count, total, share).
Usage: python tools/summarize_launches.py launches.csv > profiles/launches_rNN.txt"""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr, data = rows[hi], rows[hi + 1:]
ix = {h: i for i, h in enumerate(hdr)}
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in data:
    if r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    key = r[ix["Kernel Name"]].split("(")[0][:90]
    agg[key][0] += 1
    agg[key][1] += float(r[ix["Metric Value"]].replace(",", "")) * scale.get(r[ix["Metric Unit"]], 1e-6)
tot = sum(v[1] for v in agg.values())
print(f"# {sys.argv[1]}: {sum(v[0] for v in agg.values())} launches, {tot:.1f} ms total (ncu, serialised, cold caches)")
print(f"{'launches':>8} {'total_ms':>12} {'avg_ms':>10} {'share':>7}  kernel")
for k, (c, ms) in sorted(agg.items(), key=lambda x: -x[1][1])[:25]:
    print(f"{c:8d} {ms:12.2f} {ms / c:10.4f} {100 * ms / tot:6.2f}%  {k}")
