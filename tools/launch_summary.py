"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel count, time, share."""
import collections, csv, sys

path, title = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else "")
hdr, tot, cnt = None, collections.defaultdict(float), collections.Counter()
for r in csv.reader(open(path)):
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] == "gpu__time_duration.sum":
            k = d["Kernel Name"][:72]
            scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(d["Metric Unit"], 1e-6)
            tot[k] += float(d["Metric Value"].replace(",", "")) * scale
            cnt[k] += 1
all_ms = sum(tot.values()) or 1.0
if title:
    print(title)
print("count   total_ms   share  kernel")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{cnt[k]:5d} {v:10.3f} {100 * v / all_ms:6.1f}%  {k}")
