"""Per-CUDA-line stall samples and executed instructions from an ncu report (needs -lineinfo):
python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur, hdr, out = None, None, []


def num(x):
    try:
        return int(x)
    except ValueError:
        return 0


for r in csv.reader(io.StringIO(txt)):
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif r and r[0].isdigit() and hdr:
        out.append((num(r[4]), num(r[7]), cur, r[0], r[1].strip()[:100]))
tot = sum(o[0] for o in out) or 1
toti = sum(o[1] for o in out) or 1
print("stall samples", tot, "warp instructions", toti)
out.sort(key=lambda o: -o[0])
for o in out[:top]:
    print(f"{o[0] / tot * 100:5.1f}% stall {o[1] / toti * 100:5.1f}% inst  {o[2]}:{o[3]}  {o[4]}")
