"""Top SASS lines by warp-stall samples from an ncu report (source page), per
profiled kernel when the report holds several."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
KEY = "Warp Stall Sampling (All Samples)"
sections, cur, hdr, title = [], None, None, ""
for r in rows:
    if KEY in r:
        hdr = r
        cur = {"title": title, "hdr": hdr, "body": []}
        sections.append(cur)
    elif cur is not None and len(r) == len(hdr):
        cur["body"].append(r)
    elif len(r) == 1 or (len(r) >= 1 and r[0].startswith("Kernel")):
        title = " ".join(r)[:120]
seen = set()
for sec in sections:
    iS = sec["hdr"].index(KEY)
    body = [r for r in sec["body"] if r[iS].strip().isdigit()]
    total = sum(int(r[iS]) for r in body)
    if not total or (sec["title"], total) in seen:
        continue
    seen.add((sec["title"], total))
    body.sort(key=lambda r: -int(r[iS]))
    print(f"== {sec['title']}  total samples {total}")
    for r in body[:top]:
        print(f"{int(r[iS]) / total * 100:6.2f}%  {r[0][-5:]}  {r[1].strip()[:90]}")
