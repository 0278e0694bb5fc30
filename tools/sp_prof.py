"""Summarise an ncu report of k_sp_score: tensor activity and where the MMA
issuer / producers / epilogue stall (source-page SASS samples)."""
import csv
import subprocess
import sys

rep = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/prof_sp.ncu-rep"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, v = rows[0], rows[2]
for k in ("gpu__time_duration.sum", "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
          "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg"):
    if k in h:
        print(k, v[h.index(k)])
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
allrows = list(csv.reader(src.splitlines()))
hh, rows = allrows[1], allrows[2:]
reasons = [x for x in hh if x.startswith("stall_") and "Not Issued" not in x]
ri = [hh.index(x) for x in reasons]
tot = sum(float(r[2]) for r in rows)
mi = [n for n, r in enumerate(rows) if "UTCHMMA" in r[1]]
pi = [n for n, r in enumerate(rows) if "STTM" in r[1]]


def region(lo, hi, name, show=0):
    agg = [0.0] * len(ri)
    t = 0.0
    for n in range(lo, hi):
        for j, i in enumerate(ri):
            try:
                agg[j] += float(rows[n][i])
            except ValueError:
                pass
        t += float(rows[n][2])
    print(f"{name}: {t / tot:.3f} of samples;",
          sorted([(round(a / max(t, 1), 3), reasons[j]) for j, a in enumerate(agg)], reverse=True)[:5])
    if show:
        top = sorted([(float(rows[n][2]), n, rows[n][1][:80]) for n in range(lo, hi)], reverse=True)[:show]
        for x in top:
            print("   ", x)


region(mi[0] - 60, mi[-1] + 30, "MMA warp", 12)
region(pi[0] - 200, pi[-1] + 20, "producers", 8)
region(0, pi[0] - 200, "epilogue (+init)", 8)
