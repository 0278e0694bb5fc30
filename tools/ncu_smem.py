"""Per-source-line shared-memory wavefronts (actual vs ideal) of an ncu
report: python tools/ncu_smem.py REP."""
import csv, collections, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines())); hdr = rows[2]
iw = hdr.index('L1 Wavefronts Shared'); ii = hdr.index('L1 Wavefronts Shared Ideal')
w = collections.Counter(); wi = collections.Counter(); src = {}
for r in rows[3:]:
    if len(r) < len(hdr): continue
    try: ln = int(r[0])
    except: continue
    src[ln] = r[1][:80]
    try: w[ln] += float(r[iw] or 0); wi[ln] += float(r[ii] or 0)
    except: pass
T = sum(w.values()); print('total wavefronts', T, 'ideal', sum(wi.values()))
for ln, v in w.most_common(15): print(ln, '%.1f%%' % (100 * v / T), 'ideal %.1f%%' % (100 * wi[ln] / T), src[ln])
