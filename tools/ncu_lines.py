"""Per-source-line SASS instruction counts and stall samples from an ncu
report (`--page source --print-source cuda,sass`): the hot lines of a kernel.

    python tools/ncu_lines.py report.ncu-rep [top]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "cuda,sass", "--csv"],
                     capture_output=True, text=True).stdout
inst = collections.Counter()
samp = collections.Counter()
src = {}
path = None
hdr = None
cur = None
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        path = row[1].split("/")[-1]
        continue
    if row[0] in ("Function Name",):
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or len(row) < len(hdr):
        continue
    line = row[0]
    if row[1] and row[2] == "-":  # a cuda source line row
        cur = (path, int(line) if line.isdigit() else 0)
        src[cur] = row[1].strip()
        continue
    if cur is None:
        continue
    try:
        n = int(row[hdr.index("Instructions Executed")])
        sm = int(row[hdr.index("Warp Stall Sampling (All Samples)")])
    except ValueError:
        continue
    inst[cur] += n
    samp[cur] += sm
ti, ts = sum(inst.values()), sum(samp.values())
print(f"total instructions {ti}, samples {ts}")
for k, v in sorted(samp.items(), key=lambda t: -t[1])[:top]:
    print(f"{k[0]}:{k[1]:5d}  samp {v / ts:6.3f}  inst {inst[k] / ti:6.3f}  {src.get(k, '')[:90]}")
