"""Development aid: print an ncu --csv metrics capture as one row per launch."""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, mi, vi, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
d, names = {}, {}
for r in rows[1:]:
    d.setdefault(int(r[ii]), {})[r[mi]] = r[vi]
    names[int(r[ii])] = r[ki].split("(")[0].replace("void ", "")[-40:]
metrics = sorted({m for x in d.values() for m in x})
print("id kernel " + " ".join(m.split("__")[1][:28] if "__" in m else m for m in metrics))
for i in sorted(d):
    print(i, names[i], " ".join(d[i].get(m, "-") for m in metrics))
