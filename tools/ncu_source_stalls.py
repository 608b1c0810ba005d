"""Aggregate ncu warp-stall samples by CUDA source line for one kernel:
  ncu -i REP --page source --csv --print-source sass,cuda -k regex:NAME > src.csv
  python tools/ncu_source_stalls.py src.csv [top]"""
import collections
import csv
import sys


def main(path, top=25):
    agg, src, f = collections.Counter(), {}, None
    with open(path, errors="replace") as fh:
        for line in csv.reader(fh):
            if len(line) == 2 and line[0] in ("File Path", "File Name"):
                f = line[1].split("/")[-1]
                continue
            if len(line) > 5 and line[0].isdigit():
                try:
                    n = int(line[4] or 0)
                except ValueError:
                    continue
                key = (f, int(line[0]))
                agg[key] += n
                src[key] = line[1][:110]
    tot = max(sum(agg.values()), 1)
    for k, v in agg.most_common(top):
        print(f"{v:6d} {100 * v / tot:5.1f}% {k[0]}:{k[1]} {src[k]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
