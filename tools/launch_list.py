"""Print kernel name + duration (ns) from an ncu --csv launch list."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = None
for r in rows:
    if r and r[0] == "ID":
        h = r
        continue
    if h and len(r) == len(h):
        d = dict(zip(h, r))
        print(f'{d["Metric Value"]:>10} {d["Kernel Name"][:90]}')
