"""Per-SASS-instruction shared-memory wavefronts of one kernel in an
.ncu-rep (which loads / stores drive the shared pipe, and how many of their
wavefronts are bank-conflict excess):
    python tools/ncu_smem_lines.py rep.ncu-rep k_gather [top]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}", "--launch-count", "1",
                      "--print-source=sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
iw, ie, ii, isrc, iex = (h.index("L1 Wavefronts Shared"), h.index("L1 Wavefronts Shared Excessive"),
                         h.index("L1 Wavefronts Shared Ideal"), h.index("Source"),
                         h.index("Instructions Executed"))
data = []
for r in rows[2:]:
    if len(r) <= iw:
        continue
    try:
        w = int(r[iw] or 0)
    except ValueError:
        continue
    if w:
        data.append((w, int(r[ie] or 0), int(r[ii] or 0), int(r[iex] or 0), r[isrc].strip()))
data = sorted(set(data))  # the source page can list an instruction twice
tot = sum(d[0] for d in data) or 1
print(f"{kern}: shared wavefronts {tot}, excess {sum(d[1] for d in data)}, ideal {sum(d[2] for d in data)}")
for w, e, i, n, s in sorted(data, reverse=True)[:top]:
    print(f"{100 * w / tot:5.1f}%  wf {w:11d}  excess {e:11d}  ideal {i:11d}  exec {n:10d}  {s[:70]}")
