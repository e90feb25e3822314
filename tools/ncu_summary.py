"""Summarise an .ncu-rep: key raw metrics per kernel and the hottest SASS
segments (instruction counts and stall samples)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
kfilter = sys.argv[2] if len(sys.argv) > 2 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h = rows[0]
want = ['Kernel Name', 'gpu__time_duration.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum',
        'smsp__thread_inst_executed_per_inst_executed.ratio',
        'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum', 'l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum',
        'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_wait_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio',
        'smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio',
        'launch__registers_per_thread', 'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem']
for r in rows[2:]:
    name = r[h.index('Kernel Name')]
    if kfilter and kfilter not in name:
        continue
    print('====', name[:80])
    for w in want[1:]:
        if w in h:
            print(f"  {w:88s} {r[h.index(w)]}")
if kfilter:
    sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kfilter}",
                           "--print-source=sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(sass.splitlines()))
    hh = rows[1]
    isrc, iex, ist = hh.index('Source'), hh.index('Instructions Executed'), hh.index('Warp Stall Sampling (All Samples)')
    data = [(r[isrc].strip(), int(r[iex] or 0), int(r[ist] or 0)) for r in rows[2:]
            if len(r) > iex and r[iex].replace(',', '').isdigit() or (len(r) > iex and r[iex] == '')]
    segs, cur = [], None
    for i, (s, e, st) in enumerate(data):
        if cur and cur[2] == e:
            cur[1] = i; cur[3] += e; cur[4] += st
        else:
            cur = [i, i, e, e, st]; segs.append(cur)
    tot = sum(d[1] for d in data) or 1
    tst = sum(d[2] for d in data) or 1
    segs.sort(key=lambda x: -x[4])
    print('total warp-instr', tot)
    for a, b, e, t, st in segs[:int(sys.argv[3]) if len(sys.argv) > 3 else 15]:
        print(f"[{a:5d}-{b:5d}] n={b-a+1:3d} exec={e:9d} instr {100*t/tot:5.1f}% stall {100*st/tst:5.1f}%  {data[a][0][:40]} .. {data[b][0][:30]}")
