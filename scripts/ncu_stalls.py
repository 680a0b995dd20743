"""Per-instruction warp-stall samples from an ncu source page CSV
(ncu -i REP --page source --csv --print-source sass ...)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = {h: 0 for h in stalls}
lines = []
for r in rows[2:]:
    if len(r) < len(hdr) or not r[0].startswith("0x"):
        continue
    samp = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    ex = int(r[ix["Instructions Executed"]] or 0)
    parts = {h: int(r[ix[h]] or 0) for h in stalls}
    for h in stalls:
        tot[h] += parts[h]
    top = sorted(((v, h[6:]) for h, v in parts.items() if v), reverse=True)[:3]
    lines.append((r[ix["Address"]][-5:], r[ix["Source"]].strip()[:60], samp, ex, top))
S = sum(tot.values())
print("total samples", S, {h[6:]: v for h, v in sorted(tot.items(), key=lambda x: -x[1]) if v})
lo = int(sys.argv[2]) if len(sys.argv) > 2 else 1
for a, src, samp, ex, top in lines:
    if ex >= lo:
        print(f"{a} {samp:6d} {ex:7d}  {src:60s} {top}")
