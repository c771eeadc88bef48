"""Print the last forward's launches from gpurun_out/c2_launches.csv."""
import csv
rows = [r for r in csv.reader(open("gpurun_out/c2_launches.csv")) if len(r) > 10]
h = rows[0]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
tot = 0
for r in rows[-8:]:
    tot += float(r[vi])
    print(r[vi], "ns", r[ki][:100])
print("sum", tot)
