"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per kernel name, launches, mean device time and share of this library's
(pqkv) device time.  usage: python scripts/launch_summary.py launches.csv"""
import csv, collections, sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ik, im, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
agg = collections.OrderedDict()
for r in rows[1:]:
    if r[im] != "gpu__time_duration.sum":
        continue
    name = r[ik][:70]
    t = float(r[iv].replace(",", ""))
    unit = r[hdr.index("Metric Unit")] if "Metric Unit" in hdr else "ns"
    t = t * {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "nsecond": 1}.get(unit, 1)
    agg.setdefault(name, []).append(t)
tot = sum(sum(v) for k, v in agg.items() if "pqkv" in k)
print("# per-launch device time (ns), ncu cold-cache serialised replay: compare SHARES, not absolutes")
for k, v in agg.items():
    share = f"{100 * sum(v) / tot:5.1f}%" if "pqkv" in k and tot else "   - "
    print(f"{k:70s} n={len(v):4d} mean_ns={sum(v) / len(v):10.1f} share_of_pqkv={share}")
