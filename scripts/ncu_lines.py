"""Aggregate an ncu source page (cuda,sass) to CUDA source lines."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
cur_file = None; hdr = None; agg = {}
for r in rows:
    if not r: continue
    if r[0] == 'File Path': cur_file = r[1].split('/')[-1]; continue
    if r[0] == 'Line No': hdr = r; continue
    if hdr is None or r[0] == 'Function Name' or not r[0]: continue
    samp = hdr.index('Warp Stall Sampling (All Samples)'); ie = hdr.index('Instructions Executed')
    try:
        agg[(cur_file, int(r[0]), r[1][:95])] = [float(r[samp] or 0), float(r[ie] or 0)]
    except ValueError:
        pass
ts = sum(v[0] for v in agg.values()); ti = sum(v[1] for v in agg.values())
print(f"total samples {ts:.0f} instructions {ti:.3e}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{v[0] / ts * 100:5.1f}% samp {v[1] / ti * 100:5.1f}% inst  {k[0]}:{k[1]}  {k[2]}")
