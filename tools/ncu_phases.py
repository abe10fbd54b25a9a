"""Phase breakdown of an `ncu --page source --csv` export of a BLF kernel:
warp-stall samples and executed instructions before the first barrier (tile
staging), in the main window-row loop (the last backward branch's body) and after it."""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ci = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) == len(hdr)]
bar = next(i for i, r in enumerate(data) if "BAR.SYNC" in r[1])
addr = [int(r[0], 16) for r in data]
back = [(i, int(m.group(1), 16)) for i, r in enumerate(data) if i > bar and "BRA" in r[1]
        for m in [re.search(r"0x([0-9a-f]+)", r[1])] if m and int(m.group(1), 16) < addr[i]]
le, tgt = max(back, key=lambda t: addr[t[0]] - t[1])
ls = addr.index(tgt)
S = lambda a, b, col="# Samples": sum(int(r[ci[col]]) for r in data[a:b])
tot = S(0, len(data))
segs = {"staging (to the barrier)": (0, bar + 1), "setup + first row": (bar + 1, ls), "main loop": (ls, le + 1),
        "last row + epilogue": (le + 1, len(data))}
stalls = [h for h in hdr if h.startswith("stall_") and "Not" not in h]
for k, (a, b) in segs.items():
    d = {h: S(a, b, h) for h in stalls}
    t = max(sum(d.values()), 1)
    top = {h[6:]: round(100 * v / t, 1) for h, v in sorted(d.items(), key=lambda x: -x[1])[:6]}
    print(f"{k}: {100 * S(a, b) / tot:.1f}% of samples, {S(a, b, 'Instructions Executed')} warp instructions; {top}")
