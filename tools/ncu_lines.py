"""Per-CUDA-source-line instruction and stall shares from an .ncu-rep
(needs -lineinfo): python tools/ncu_lines.py rep.ncu-rep [kernel-regex] [top]"""
import csv, subprocess, sys
rep = sys.argv[1]
kf = sys.argv[2] if len(sys.argv) > 2 else None
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
if kf:
    cmd += ["--kernel-name", f"regex:{kf}", "--launch-count", "1"]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
res, fname = [], None
for r in csv.reader(out.splitlines()):
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if len(r) > 8 and r[0] not in ("", "Line No") and r[0].isdigit():
        try:
            st, ex = int(r[4]), int(r[7])
        except ValueError:
            continue
        if ex or st:
            res.append((fname, int(r[0]), ex, st, r[1].strip()[:80]))
tot = sum(x[2] for x in res) or 1
tst = sum(x[3] for x in res) or 1
print(f"total instr {tot}  stall samples {tst}")
for f, ln, ex, st, src in sorted(res, key=lambda x: -(x[2] / tot + x[3] / tst))[:top]:
    print(f"{f}:{ln:<5d} instr {100*ex/tot:5.1f}%  stall {100*st/tst:5.1f}%  {src}")
