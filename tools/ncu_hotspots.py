"""Top SASS lines by warp-stall samples from an ncu report (source page)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
iS = hdr.index("Warp Stall Sampling (All Samples)")
body = [r for r in rows[2:] if len(r) == len(hdr)]
total = sum(int(r[iS]) for r in body)
body.sort(key=lambda r: -int(r[iS]))
print(f"total samples {total}")
for r in body[:top]:
    print(f"{int(r[iS]) / total * 100:6.2f}%  {r[0][-5:]}  {r[1].strip()[:90]}")
