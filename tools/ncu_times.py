import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = [r for r in rows if r and r[0] == "ID"][0]
for r in rows:
    if len(r) == len(h) and r[0] != "ID" and r[h.index("Metric Name")] == "gpu__time_duration.sum":
        print(r[h.index("Kernel Name")][:60], r[h.index("Metric Value")])
