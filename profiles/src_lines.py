"""Per-CUDA-source-line warp-stall samples and executed warp instructions of one function from
`ncu --page source --csv --print-source cuda,sass` (interleaved).  usage: src_lines.py CSV[.gz] FUNC_SUBSTR [top]"""
import collections, csv, gzip, sys

path, func = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
op = gzip.open if path.endswith(".gz") else open
cur_file = cur_func = cur_line = None
src = {}
samp, inst = collections.Counter(), collections.Counter()
hdr = None
with op(path, "rt") as f:
    for r in csv.reader(f):
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]; continue
        if r[0] == "Function Name":
            cur_func = r[1]; continue
        if r[0] == "Line No":
            hdr = r; continue
        if hdr is None or func not in (cur_func or ""):
            continue
        if r[0].strip():
            cur_line = (cur_file, r[0]); src[cur_line] = r[1].strip()[:90]; continue
        try:
            samp[cur_line] += int(r[hdr.index("Warp Stall Sampling (All Samples)")])
            inst[cur_line] += int(r[hdr.index("Instructions Executed")])
        except (ValueError, IndexError):
            pass
ts, ti = sum(samp.values()) or 1, sum(inst.values()) or 1
print(f"{func}: samples {ts}, warp instructions {ti}")
for k, v in sorted(inst.items(), key=lambda kv: -kv[1])[:top]:
    print(f"inst {100*v/ti:5.1f}%  samp {100*samp[k]/ts:5.1f}%  {k[0]}:{k[1]}  {src.get(k, '')}")
