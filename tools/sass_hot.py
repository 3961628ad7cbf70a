"""Top SASS instructions by stall samples from `ncu --page source --csv --print-source sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr) and r[0].startswith("0x")]
iS = hdr.index("Warp Stall Sampling (All Samples)")
iE = hdr.index("Instructions Executed")
iSrc = hdr.index("Source")
f = lambda x: float(x) if x not in ("", "-") else 0.0  # noqa: E731
tot = sum(f(r[iS]) for r in data) or 1.0
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
for r in sorted(data, key=lambda r: -f(r[iS]))[:n]:
    print(f"{f(r[iS]) / tot * 100:5.1f}% exec={f(r[iE]):>9.0f} {r[0][-5:]} {r[iSrc].strip()[:100]}")
