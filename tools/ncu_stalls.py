"""Warp-stall reasons and instruction mix of one launch in an ncu report (run HERE, no GPU):
    python tools/ncu_stalls.py report.ncu-rep LAUNCH_INDEX"""
import csv, subprocess, sys, io
rep, idx = sys.argv[1], int(sys.argv[2])
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass', '-k', 'regex:wl_gemv',
                      '--launch-skip', str(idx), '--launch-count', '1'], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
his = [i for i, r in enumerate(rows) if 'Address' in r and 'Source' in r]
hdr = rows[his[0]]
data = rows[his[0] + 1:(his[1] if len(his) > 1 else None)]
def num(v):
    try: return float(v)
    except: return 0.0
iS = hdr.index('Source'); iW = hdr.index('Warp Stall Sampling (All Samples)'); iE = hdr.index('Instructions Executed')
stall = [h for h in hdr if h.startswith('stall_')]
from collections import Counter
tot = sum(num(r[iW]) for r in data if len(r) == len(hdr))
reasons = Counter(); ex = Counter(); exall = 0
for r in data:
    if len(r) != len(hdr): continue
    toks = r[iS].split()
    if not toks: continue
    op = toks[1] if toks[0].startswith('@') else toks[0]
    ex[op.split('.')[0]] += num(r[iE]); exall += num(r[iE])
    for h in stall: reasons[h] += num(r[hdr.index(h)])
print(f"launch {idx}: samples {tot:.0f}, warp-instrs executed {exall:.0f}")
print("  top ops:", ", ".join(f"{k} {100*v/exall:.1f}%" for k, v in ex.most_common(10)))
print("  stalls:", ", ".join(f"{k[6:]} {100*v/tot:.1f}%" for k, v in reasons.most_common(9)))
