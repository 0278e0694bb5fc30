"""Per-source-line warp-stall samples and instruction counts of an ncu
report (--set full --import-source on): python tools/ncu_lines.py REP [N]."""
import csv, collections, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[2]
iS = hdr.index('Warp Stall Sampling (All Samples)'); iI = hdr.index('Instructions Executed')
reasons = [h for h in hdr if h.startswith('stall_') and 'Not' not in h]
by = collections.Counter(); byi = collections.Counter(); src = {}; per = collections.defaultdict(collections.Counter)
for r in rows[3:]:
    if len(r) < len(hdr): continue
    try: ln = int(r[0])
    except: continue
    src[ln] = r[1][:80]
    try:
        by[ln] += float(r[iS] or 0); byi[ln] += float(r[iI] or 0)
        for h in reasons: per[ln][h] += float(r[hdr.index(h)] or 0)
    except: pass
tot = sum(by.values()); ti = sum(byi.values())
print('samples', tot, 'instr', ti)
for ln, v in by.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    top = ' '.join('%s=%.1f' % (k[6:], 100 * x / tot) for k, x in per[ln].most_common(2))
    print(ln, '%.1f%%' % (100 * v / tot), 'i%.1f%%' % (100 * byi[ln] / ti), top, '|', src.get(ln))
