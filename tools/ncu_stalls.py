"""Stall-reason totals for the SASS lines attributed to a source-line range:
python tools/ncu_stalls.py src.csv FILE LO HI   (from `ncu -i X --page source --csv --print-source cuda,sass`)."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
fname, lo, hi = sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
hdr = None; cur_file = None; cur_line = None
tot = collections.Counter(); alltot = collections.Counter()
for r in rows:
    if not r: continue
    if r[0] == "File Path": cur_file = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None: continue
    if r[0].isdigit(): cur_line = int(r[0]); continue
    if len(r) > 2 and r[2].startswith("0x"):
        for k, v in zip(hdr, r):
            if k.startswith("stall_") and "Not Issued" not in k:
                try: x = int(v or 0)
                except ValueError: continue
                alltot[k] += x
                if cur_file == fname and lo <= (cur_line or -1) <= hi: tot[k] += x
s = sum(tot.values()) or 1; S = sum(alltot.values()) or 1
print(f"range share of all samples: {100*s/S:.1f}%")
for k, v in tot.most_common(): print(f"{k:28s} {100*v/s:5.1f}%")
