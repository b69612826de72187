"""Hot SASS instructions of one kernel in an ncu report (instructions executed, stall
samples), to read a kernel's inner loops here without a GPU.

  python scripts/ncu_sass_hot.py <report.ncu-rep> [top=40]
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--launch-count", "1"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
rows = list(csv.reader(lines[1:]))
h = rows[0]
ia, isrc, ismp, iex = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), \
    h.index("Instructions Executed")
data = []
for i, r in enumerate(rows[1:]):
    try:
        data.append((i, r[isrc].strip(), int(r[ismp] or 0), int(r[iex] or 0)))
    except (ValueError, IndexError):
        pass
tot_s = sum(d[2] for d in data)
tot_e = sum(d[3] for d in data)
print(f"instructions executed {tot_e:,}  stall samples {tot_s:,}  sass lines {len(data)}")
# coarse profile: blocks of 32 consecutive instructions
print("-- by block of 32 SASS lines: first line, inst executed, samples")
for b in range(0, len(data), 32):
    blk = data[b:b + 32]
    e = sum(d[3] for d in blk)
    s = sum(d[2] for d in blk)
    if e > 0.01 * tot_e or s > 0.01 * tot_s:
        print(f"{b:5d} {e / tot_e * 100:6.1f}% inst {s / tot_s * 100:6.1f}% smp  {blk[0][1][:60]}")
print("-- top instructions by samples")
for d in sorted(data, key=lambda d: -d[2])[:top]:
    print(f"{d[0]:5d} smp {d[2]:7d} ex {d[3]:10d}  {d[1][:80]}")
