"""Stall-reason breakdown of an ncu report, grouped by SASS opcode class,
excluding the mbarrier wait loops (reported separately)."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
body = [r for r in rows[2:] if len(r) == len(hdr)]
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
idx = {h: hdr.index(h) for h in reasons}
by_op = collections.defaultdict(lambda: collections.Counter())
tot = collections.Counter()
for i, r in enumerate(body):
    op = r[1].strip().split()[0] if r[1].strip() else "?"
    if op.startswith("@"):
        op = r[1].strip().split()[1]
    op = op.split(".")[0]
    # attribute the try-wait loop (TRYWAIT + BRA) to "mbar_wait"
    if op == "BRA" and i > 0 and "TRYWAIT" in body[i - 2][1] + body[i - 1][1]:
        op = "mbar_wait"
    if op == "SYNCS":
        op = "mbar_wait"
    for h in reasons:
        v = int(float(r[idx[h]] or 0))
        by_op[op][h] += v
        tot[h] += v
grand = sum(tot.values())
print("all samples", grand)
print("by reason:", ", ".join(f"{k[6:]} {v / grand * 100:.1f}%" for k, v in tot.most_common(8)))
ops = sorted(by_op.items(), key=lambda kv: -sum(kv[1].values()))
for op, c in ops[:18]:
    s = sum(c.values())
    print(f"{op:12s} {s / grand * 100:5.1f}%  " +
          ", ".join(f"{k[6:]} {v / s * 100:.0f}%" for k, v in c.most_common(3)))
