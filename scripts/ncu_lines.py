"""Aggregate an ncu 'cuda,sass' source export by CUDA source line (stall samples, instructions, local ops)."""
import csv, gzip, sys, collections
path = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
rows = list(csv.reader(gzip.open(path, 'rt') if path.endswith('.gz') else open(path)))
hdr = None; f = None; line = None
agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0, 0.0])
for r in rows:
    if r and r[0] == 'File Path': f = r[1].split('/')[-1]; continue
    if r and r[0] == 'Line No': hdr = r; continue
    if not hdr or len(r) < 5: continue
    if r[0] != '': line = (f, r[0], r[1][:110]); continue
    d = dict(zip(hdr[2:], r[2:]))
    try:
        ie = float(d.get('Instructions Executed', '0') or 0); ss = float(d.get('Warp Stall Sampling (All Samples)', '0') or 0)
    except ValueError:
        continue
    a = agg[line]; a[0] += ie; a[3] += ss
    if 'STL' in r[3]: a[1] += ie
    if 'LDL' in r[3]: a[2] += ie
T = sum(v[3] for v in agg.values()) or 1
print(f"samples {T:.0f}; instructions {sum(v[0] for v in agg.values()):.0f}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][3])[:top]:
    print(f"{100 * v[3] / T:5.1f}% {int(v[0]):9d} {k[0]}:{k[1]} {k[2]}")
