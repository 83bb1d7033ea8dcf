"""Summarise an ncu DRAM capture of scripts/fused_step.py (one or more fused preprocess +
count steps) into the committed per-kernel table and profiles/traffic.json.

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        --clock-control none --csv --log-file gpurun_out/X.csv python scripts/fused_step.py 26 2
    python scripts/step_profile.py gpurun_out/X.csv profiles/r02_step_dram_s26.md [label]

The LAST step of the capture is summarised (the first warms the pools).  Kernels from the
first preprocessing kernel (k_degree_hist) up to the first count kernel are the preprocess
phase; the rest are the count phase.  ncu times are serialised and cold-cache: use shares
and bytes, not absolute times, against the bench's CUDA-event numbers."""
import collections
import csv
import json
import os
import sys

PEAK = 6522.1
try:
    PEAK = float(json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"])
except (OSError, KeyError, ValueError):
    pass

src, out = sys.argv[1], sys.argv[2]
label = sys.argv[3] if len(sys.argv) > 3 else os.path.basename(src)
rows = [r for r in csv.reader(open(src)) if len(r) > 10]
h = rows[0]
ki, mi, vi, idi = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
per = collections.OrderedDict()
for r in rows[1:]:
    per.setdefault(int(r[idi]), {"name": r[ki].split("(")[0].replace("void ", "").replace("unnamed>::", "")})
    per[int(r[idi])][r[mi]] = float(r[vi].replace(",", ""))
launches = [per[k] for k in sorted(per)]
starts = [i for i, d in enumerate(launches) if d["name"].startswith("k_degree_hist")]
step = launches[starts[-1]:] if starts else launches
first_count = next((i for i, d in enumerate(step) if d["name"].startswith(("k_range_init", "k_classify"))), len(step))
phases = {"preprocess": step[:first_count], "count": step[first_count:]}


def agg(ks):
    t = collections.OrderedDict()
    for d in ks:
        a = t.setdefault(d["name"], {"n": 0, "ms": 0.0, "rd": 0.0, "wr": 0.0})
        a["n"] += 1
        a["ms"] += d.get("gpu__time_duration.sum", 0) / 1e6
        a["rd"] += d.get("dram__bytes_read.sum", 0)
        a["wr"] += d.get("dram__bytes_write.sum", 0)
    return t


lines = [f"# One fused step (preprocess + count), DRAM traffic per kernel (ncu) — {label}", "",
         f"Source: `{src}` (last step of `scripts/fused_step.py`); peak {PEAK} GB/s (MEASURED_PEAKS.json). "
         "ncu times are serialised / cold-cache: compare shares and bytes with bench.py's CUDA-event times.", ""]
summary = {}
for ph, ks in phases.items():
    t = agg(ks)
    tot_ms = sum(a["ms"] for a in t.values())
    tot_b = sum(a["rd"] + a["wr"] for a in t.values())
    summary[ph] = {"ms": tot_ms, "bytes": tot_b}
    lines += [f"## {ph}: {tot_ms:.1f} ms, {tot_b / 1e9:.1f} GB, {tot_b / max(tot_ms, 1e-9) / 1e6:.0f} GB/s "
              f"({tot_b / max(tot_ms, 1e-9) / 1e6 / PEAK:.2f} of peak)", "",
              "| kernel | launches | ms | share | DRAM read GB | DRAM write GB | GB/s | frac of peak |",
              "|---|---|---|---|---|---|---|---|"]
    for name, a in sorted(t.items(), key=lambda kv: -kv[1]["ms"]):
        if a["ms"] < 0.005:
            continue
        gbs = (a["rd"] + a["wr"]) / a["ms"] / 1e6 if a["ms"] else 0
        lines.append(f"| `{name}` | {a['n']} | {a['ms']:.2f} | {100 * a['ms'] / tot_ms:.1f}% | "
                     f"{a['rd'] / 1e9:.2f} | {a['wr'] / 1e9:.2f} | {gbs:.0f} | {gbs / PEAK:.2f} |")
    lines.append("")
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
tj = "profiles/traffic.json"
try:
    data = json.load(open(tj))
except (OSError, ValueError):
    data = {}
data["rmat_s26_ef16_seed0"] = {
    "dram_bytes_per_count": summary["count"]["bytes"],
    "count_kernels_ms_under_ncu": summary["count"]["ms"],
    "dram_bytes_per_preprocess": summary["preprocess"]["bytes"],
    "preprocess_kernels_ms_under_ncu": summary["preprocess"]["ms"],
    "source": f"{out} ({label}): ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,"
              "gpu__time_duration.sum python scripts/fused_step.py 26 2, last step",
}
json.dump(data, open(tj, "w"), indent=1)
