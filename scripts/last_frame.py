"""Print the kernel launches (name, us) of the last forward frame in an ncu --csv launch list."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ik, iv = h.index("Kernel Name"), h.index("Metric Value")
fr = [(r[ik].split("(")[0].replace("geer::<unnamed>::", "").replace("void geer::", "")[-48:], float(r[iv].replace(",", "")) / 1e3)
      for r in rows[hi + 1:] if len(r) == len(h)]
start = max(i for i, x in enumerate(fr) if "k_preprocess" in x[0])
tot = 0.0
for name, us in fr[start:]:
    if "k_sum_i32" in name:
        continue
    tot += us
    print(f"{us:9.1f}  {name}")
print(f"{tot:9.1f}  total")
