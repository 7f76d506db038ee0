"""Summarise an ncu launch list (gpu__time_duration.sum per launch) of `bench.py --steps 1
--warmup 1`: per-kernel totals of the TIMED step (the second occurrence of k_tag starts it)."""
import collections
import csv
import sys


def main(path, out=None):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    ui = hdr.index("Metric Unit")
    launches = [(r[ki], float(r[vi].replace(",", "")) * (1e-3 if r[ui] in ("ns", "nsecond") else 1.0))
                for r in rows[1:] if r[mi] == "gpu__time_duration.sum"]
    starts = [i for i, (k, _) in enumerate(launches) if k.startswith("k_tag")]
    timed = launches[starts[1]:] if len(starts) > 1 else launches
    tot = collections.defaultdict(lambda: [0, 0.0])
    for k, us in timed:
        name = k.split("(")[0]
        tot[name][0] += 1
        tot[name][1] += us
    T = sum(v[1] for v in tot.values())
    lines = ["kernel,launches,total_us,share"]
    for k, (n, us) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{k},{n},{us:.1f},{us / T:.4f}")
    lines.append(f"TOTAL,{sum(v[0] for v in tot.values())},{T:.1f},1.0")
    txt = "\n".join(lines)
    if out:
        open(out, "w").write(txt + "\n")
    print(txt)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
