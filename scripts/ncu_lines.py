"""Top CUDA source lines of an ncu report by warp-stall samples (needs -lineinfo and
--import-source on).  usage: ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
lines = []
cur_file = ""
hdr = None
for r in rows:
    if r and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0]:
        d = dict(zip(hdr, r))
        try:
            s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
            ins = int(d.get("Instructions Executed", "0") or 0)
        except ValueError:
            continue
        lines.append((s, ins, cur_file, r[0], r[1][:90]))
tot = sum(x[0] for x in lines) or 1
toti = sum(x[1] for x in lines) or 1
for s, ins, f, ln, src in sorted(lines, reverse=True)[:top]:
    print(f"{100 * s / tot:5.1f}% st {100 * ins / toti:5.1f}% in  {f}:{ln:>5}  {src}")
