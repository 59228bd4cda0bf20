"""Summarise an ncu --csv launch list: per-kernel time/bytes for the last decode iteration."""
import csv, collections, io, sys
path = sys.argv[1]
marker = sys.argv[2] if len(sys.argv) > 2 else "embed_kernel"
txt = open(path).read().splitlines()
start = [i for i, l in enumerate(txt) if l.startswith('"ID"')][0]
rows = list(csv.DictReader(io.StringIO("\n".join(txt[start:]))))
by = collections.OrderedDict()
for r in rows:
    by.setdefault(r["ID"], {"name": r["Kernel Name"]})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
ks = list(by.values())
idx = [i for i, k in enumerate(ks) if marker in k["name"]]
last = ks[idx[-1]:] if idx else ks
agg = collections.OrderedDict()
for k in last:
    n = k["name"].split("(")[0].replace("void ", "")[:48]
    a = agg.setdefault(n, [0, 0.0, 0.0])
    a[0] += 1; a[1] += k.get("gpu__time_duration.sum", 0)
    a[2] += k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0)
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':48s} {'n':>4s} {'total_us':>9s} {'avg_us':>8s} {'share':>6s} {'MB/launch':>9s} {'GB/s':>7s}")
for k, (n, t, b) in agg.items():
    print(f"{k:48s} {n:4d} {t/1e3:9.1f} {t/n/1e3:8.2f} {t/tot:6.1%} {b/n/1e6:9.2f} {b/t if t else 0:7.0f}")
print(f"total {tot/1e3:.1f} us over {len(last)} launches")
