"""Development aid: per-kernel table of an `ncu --metrics ... --csv` log (kernels >= 0.5 ms)."""
import collections
import csv
import sys

lines = open(sys.argv[1]).read().splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
by = collections.OrderedDict()
for r in csv.DictReader(lines[start:]):
    k = (r["ID"], r["Kernel Name"].split("(")[0].replace("void unnamed>::", ""))
    by.setdefault(k, {})[r["Metric Name"]] = r["Metric Value"]
for (i, k), m in by.items():
    t = float(m["gpu__time_duration.sum"].replace(",", "")) / 1e6
    if t < 0.5:
        continue
    print(f"{k[:30]:30s} {t:8.2f} ms", " ".join(f"{n.split('__')[1][:40]}={v}" for n, v in m.items()
                                                if n != "gpu__time_duration.sum"))
