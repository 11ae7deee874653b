"""Aggregate an ncu --csv launch list by kernel name."""
import csv
import collections
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] == "gpu__time_duration.sum":
            name = d["Kernel Name"].split("(")[0][:70]
            tot[name] += float(d["Metric Value"]) / 1e3
            cnt[name] += 1
allt = sum(tot.values())
print(f"total {allt:.1f} us over {sum(cnt.values())} launches")
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:30]:
    print(f"{v:10.1f} us {100*v/allt:5.1f}% {cnt[k]:6d}  {v/cnt[k]:8.2f} us/launch  {k}")
