"""Group the per-line profile of one kernel by source-line ranges:
python tools/ncu_phases.py rep kernel file.cu name:lo-hi name:lo-hi ..."""
import csv, subprocess, sys
rep, kf, src = sys.argv[1], sys.argv[2], sys.argv[3]
ranges = []
for a in sys.argv[4:]:
    n, r = a.split(":"); lo, hi = r.split("-"); ranges.append((n, int(lo), int(hi)))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", f"regex:{kf}", "--launch-count", "1"], capture_output=True, text=True).stdout
agg, fname = {}, None
tot = tst = 0
for r in csv.reader(out.splitlines()):
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if len(r) > 8 and r[0].isdigit():
        try:
            st, ex = int(r[4]), int(r[7])
        except ValueError:
            continue
        ln = int(r[0]); name = "other:" + fname
        if fname == src:
            for n, lo, hi in ranges:
                if lo <= ln <= hi: name = n; break
        elif fname.startswith("sm_100_rt"):
            name = "f32x2 intrinsics"
        a = agg.setdefault(name, [0, 0]); a[0] += ex; a[1] += st; tot += ex; tst += st
for n, (ex, st) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{n:28s} instr {100*ex/tot:5.1f}%  stall {100*st/tst:5.1f}%")
