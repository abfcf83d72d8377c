"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel launches / mean duration / share of the listed pipeline time.
usage: launch_summary.py launches.csv OUT.txt "header comment" """
import collections
import csv
import sys

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
h = rows[0]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
setup_names = ("noise_blur_rows", "blur_cols", "compose")
t = collections.OrderedDict()
setup = collections.OrderedDict()
for r in rows[1:]:
    name = r[ki].split("(")[0]
    us = float(r[vi].replace(",", "")) / 1e3
    (setup if any(s in name for s in setup_names) else t).setdefault(name, []).append(us)
total = sum(sum(v) for v in t.values())
out = ["# launch list (ncu --metrics gpu__time_duration.sum --clock-control none, cold-cache, serialised)",
       "# " + sys.argv[3], "# kernel, launches, mean_us, share_of_listed_time"]
for k, v in t.items():
    out.append("%s, %d, %.1f, %.3f" % (k, len(v), sum(v) / len(v), sum(v) / total))
out.append("# setup, untimed (on-device input generation, once per run): " +
           "; ".join("%s %.1f us" % (k, sum(v)) for k, v in setup.items()))
open(sys.argv[2], "w").write("\n".join(out) + "\n")
print("\n".join(out))
