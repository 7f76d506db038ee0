"""Warp-stall samples per CUDA source line from `ncu -i X.ncu-rep --page source --csv
--print-source cuda,sass` (interleaved source/SASS listing)."""
import collections
import csv
import sys


def main(path, top=25):
    cur_file, cur_line, cur_src = None, None, ""
    agg = collections.Counter()
    src = {}
    hdr = None
    for r in csv.reader(open(path)):
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 5:
            continue
        if r[0].strip():
            cur_line, cur_src = r[0], r[1]
            src[(cur_file, cur_line)] = cur_src.strip()[:100]
        try:
            n = int(r[4])
        except ValueError:
            continue
        agg[(cur_file, cur_line)] += n
    tot = sum(agg.values())
    print("total samples", tot)
    for (f, ln), n in agg.most_common(top):
        print(f"{100 * n / tot:5.1f}%  {f}:{ln}  {src.get((f, ln), '')}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
