"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list into markdown."""
import collections
import csv
import sys

src, dst, title = sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else ""
rows = [r for r in csv.reader(open(src)) if len(r) > 5]
h = rows[0]
i_name, i_val, i_unit = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
agg = collections.OrderedDict()
for r in rows[1:]:
    name = r[i_name].split("(")[0].replace("void ", "").strip()
    v = float(r[i_val].replace(",", "")) * scale[r[i_unit]]
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(a[1] for a in agg.values())
with open(dst, "w") as f:
    f.write(f"# {title}\n\nncu --metrics gpu__time_duration.sum --clock-control none. Per-launch device times are "
            "cold-cache and serialised: compare SHARES, not absolutes.\n\n"
            "| kernel | launches | total us | mean us | share |\n|---|---|---|---|---|\n")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        f.write(f"| `{k}` | {c} | {t:.1f} | {t / c:.1f} | {100 * t / tot:.1f}% |\n")
print(open(dst).read())
