"""Split a kernel's SASS (ncu --page source --print-source sass CSV) at its
barriers / mbarrier waits and print warp-stall samples and executed
instructions per region.  usage: ncu_sass_regions.py REPORT KERNEL_REGEX"""
import csv
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kre, "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
iS, iE = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")


def num(x):
    try:
        return float(x or 0)
    except ValueError:
        return 0.0


seen, lst = set(), []
for r in rows[2:]:
    if len(r) < len(h) or r[0] in seen or not r[0].startswith("0x"):
        continue
    seen.add(r[0])
    lst.append(r)
tot_s = sum(num(r[iS]) for r in lst)
tot_e = sum(num(r[iE]) for r in lst)
print(f"samples {tot_s:.0f}  warp-instructions {tot_e:.3e}")
cut, s, e, n = lst[0][0][-5:], 0.0, 0.0, 0
for r in lst:
    op = r[1]
    if ("BAR.SYNC" in op or "TRYWAIT" in op) and n:
        print(f"{cut:>6} .. {r[0][-5:]:>6}  {n:5d} instr  samples {s:7.0f} ({s / tot_s * 100:4.1f}%)  exec {e / tot_e * 100:4.1f}%")
        cut, s, e, n = r[0][-5:], 0.0, 0.0, 0
    s += num(r[iS])
    e += num(r[iE])
    n += 1
print(f"{cut:>6} .. end     {n:5d} instr  samples {s:7.0f} ({s / tot_s * 100:4.1f}%)  exec {e / tot_e * 100:4.1f}%")
