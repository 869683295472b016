"""Per-source-line warp-stall samples from `ncu -i X --page source --csv --print-source cuda,sass`."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cur_file = None; hdr = None
lines = []; sass = []; cur = None
for r in rows:
    if not r: continue
    if r[0] == "File Path": cur_file = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) < 6: continue
    si = 4
    try: s = int(r[si] or 0)
    except ValueError: continue
    if r[0].isdigit():
        cur = f"{cur_file}:{r[0]} {r[1].strip()[:80]}"
        lines.append((s, cur))
    elif r[2].startswith("0x"):
        sass.append((s, r[3].strip(), cur))
tot = sum(s for s, _ in lines) or 1
print("total samples", tot)
for s, k in sorted(lines, reverse=True)[:top]: print(f"{100*s/tot:5.1f}% {k}")
print("--- top SASS")
for s, ins, ln in sorted(sass, reverse=True)[:top // 2]: print(f"{100*s/tot:5.1f}% {ins[:50]:50s} | {(ln or '')[:70]}")
