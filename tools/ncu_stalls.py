"""Top warp-stall SASS lines per kernel from `ncu --page source --csv --print-source sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = [r[1][:70], None, []]
        blocks.append(cur)
    elif r and r[0] == "Address" and cur:
        cur[1] = r
    elif r and r[0].startswith("0x") and cur:
        cur[2].append(r)
seen = set()
for name, hdr, data in blocks:
    if name in seen or hdr is None:
        continue
    seen.add(name)
    ai, si = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
    d = [(int(r[si] or 0), r[ai].strip(), r[0][-5:]) for r in data]
    tot = sum(x[0] for x in d)
    print(f"KERNEL {name}  samples={tot} instr={len(d)}")
    for s, src, a in sorted(d, reverse=True)[:top]:
        print(f"  {s:7d} {100.0 * s / max(tot, 1):5.1f}% {a} {src[:90]}")
