"""Per-opcode instruction counts and warp-stall samples of one kernel from an
ncu SASS source export:
  ncu -i REP --page source --csv --print-source sass -k regex:NAME > sass.csv
  python tools/ncu_sass_ops.py sass.csv [kernel-substring] [top]
Sections of device functions called by the kernel (noinline) are included."""
import collections
import csv
import sys


def main(path, top=30):
    rows = list(csv.reader(open(path, errors="replace")))
    ops, samp, by_fn = collections.Counter(), collections.Counter(), collections.Counter()
    hdr, fn, seen = None, None, set()
    tot = stot = 0
    for r in rows:
        if r and r[0] == "Kernel Name":
            fn = r[1].split("(")[0]
            hdr = None
            continue
        if r and r[0] == "Address":
            hdr = r
            ie, iw = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        if (fn, r[0]) in seen:  # ncu repeats sections per captured launch
            continue
        seen.add((fn, r[0]))
        try:
            n = int(r[ie].replace(",", "") or 0)
            s = int(r[iw].replace(",", "") or 0)
        except ValueError:
            continue
        t = r[1].split()
        if not t:
            continue
        op = t[1] if t[0].startswith("@") and len(t) > 1 else t[0]
        op = op.split(".")[0]
        ops[op] += n
        samp[op] += s
        by_fn[fn] += n
        tot += n
        stot += s
    print(f"warp instructions {tot}, stall samples {stot}")
    for f, n in by_fn.most_common():
        print(f"  {f}: {n} ({100 * n / max(tot, 1):.1f}%)")
    for k, v in ops.most_common(top):
        print(f"{k:12s} {v:12d} {100 * v / max(tot, 1):5.1f}%  stall {100 * samp[k] / max(stot, 1):5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
