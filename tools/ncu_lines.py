"""Per-source-line executed instructions of one ncu report (needs --import-source).
Usage: python tools/ncu_lines.py report.ncu-rep n_blocks [top]"""
import csv
import io
import subprocess
import sys

rep, nblk = sys.argv[1], float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 50
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
out, cur = [], None
for r in csv.reader(io.StringIO(txt)):
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) < 9 or r[0] in ("Line No", "Function Name") or r[0] == "":
        continue
    try:
        inst, smp = int(r[7]), int(r[6])
    except ValueError:
        continue
    out.append((inst, smp, cur, r[0], r[1][:95]))
tot = sum(o[0] for o in out)
ts = sum(o[1] for o in out) or 1
print(f"total: {tot * 32 / nblk:.1f} thread-instr slots per block; samples {ts}")
for o in sorted(out, reverse=True)[:top]:
    print(f"{o[0] * 32 / nblk:7.1f}  {o[1] / ts * 100:5.1f}%smp  {o[2]}:{o[3]}  {o[4]}")
