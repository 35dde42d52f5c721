"""Top SASS instructions by warp-stall samples for one kernel of an ncu report (source page).

    python scripts/ncu_hot.py report.ncu-rep "<kernel substring>" [top]
"""
import csv
import io
import subprocess
import sys

rep, want = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks, cur = [], None
for line in out.splitlines():
    if line.startswith('"Kernel Name"'):
        cur = [line]
        blocks.append(cur)
    elif cur is not None:
        cur.append(line)
for b in blocks:
    if want not in b[0]:
        continue
    rows = list(csv.reader(io.StringIO("\n".join(b[1:]))))
    hdr = rows[0]
    si, ai = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
    body = [r for r in rows[1:] if len(r) == len(hdr)]
    tot = sum(int(r[ai] or 0) for r in body)
    print(b[0][:120], "total samples", tot)
    for k, r in sorted(enumerate(body), key=lambda kr: -int(kr[1][ai] or 0))[:top]:
        ctx = " || ".join(x[si].strip()[:40] for x in body[max(0, k - 2):k])
        print(f"{int(r[ai]):7d} {100 * int(r[ai]) / max(tot, 1):5.1f}%  {r[si].strip()[:70]:70s}  <- {ctx}")
    break
