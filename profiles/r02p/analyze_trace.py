"""Summarise an AGIPC_TRACE file: the last traced call sequence starting at `first` (default
k_tag): per launch start, duration, idle gap before it (on any stream) and host submit offset."""
import sys
path = sys.argv[1]
first = sys.argv[2] if len(sys.argv) > 2 else "k_tag"
recs = []
for line in open(path):
    if line.startswith("#"):
        continue
    parts = line.split()
    name, (s, t0, t1, hs) = " ".join(parts[:-4]), parts[-4:]
    recs.append((name, s, float(t0), float(t1), float(hs)))
starts = [i for i, r in enumerate(recs) if r[0] == first]
seq = recs[starts[-2]:starts[-1]] if len(starts) > 1 else recs[starts[-1]:]
if len(starts) > 1:  # the last complete call before the final one
    pass
base, hbase = seq[0][2], seq[0][4]
busy_end = base
tot_gap = tot_k = 0.0
print(f"{'kernel':40s} {'start':>9s} {'dur':>8s} {'gap':>7s} {'host':>9s} stream")
for name, s, t0, t1, hs in seq:
    if name.startswith("@"):  # host-time marker
        print(f"{name[:40]:40s} {'':>9s} {'':>8s} {'':>7s} {hs-hbase:9.1f} host")
        continue
    gap = max(0.0, t0 - busy_end)
    tot_gap += gap
    tot_k += t1 - t0
    busy_end = max(busy_end, t1)
    print(f"{name[:40]:40s} {t0-base:9.1f} {t1-t0:8.1f} {gap:7.1f} {hs-hbase:9.1f} {s[-4:]}")
print(f"span {busy_end-base:.1f} us, sum of kernel durations {tot_k:.1f} us, idle gaps {tot_gap:.1f} us, "
      f"launches {len(seq)}")
