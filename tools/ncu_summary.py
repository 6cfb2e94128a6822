"""Markdown summary of an ncu report: launch config, duration, IPC, occupancy,
DRAM traffic, pipe utilisation and the top stall lines (needs -lineinfo).
usage: python tools/ncu_summary.py report.ncu-rep [title] > profiles/x.md"""
import csv, io, subprocess, sys, collections

rep = sys.argv[1]
title = sys.argv[2] if len(sys.argv) > 2 else rep
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
m = dict(zip(hdr, vals))
u = dict(zip(hdr, units))
want = ["Kernel Name", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "gpu__time_duration.sum", "sm__cycles_elapsed.avg",
        "smsp__inst_executed.sum", "sm__inst_executed.avg.per_cycle_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__average_warp_latency_per_inst_issued.ratio",
        "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
        "smsp__warp_issue_stalled_short_scoreboard_per_warp_active.pct",
        "smsp__warp_issue_stalled_wait_per_warp_active.pct",
        "smsp__warp_issue_stalled_math_pipe_throttle_per_warp_active.pct",
        "smsp__warp_issue_stalled_barrier_per_warp_active.pct",
        "smsp__warp_issue_stalled_membar_per_warp_active.pct",
        "smsp__warp_issue_stalled_no_instruction_per_warp_active.pct",
        "smsp__warp_issue_stalled_mio_throttle_per_warp_active.pct",
        "smsp__warp_issue_stalled_lg_throttle_per_warp_active.pct",
        "smsp__warp_issue_stalled_not_selected_per_warp_active.pct",
        "smsp__warp_issue_stalled_selected_per_warp_active.pct"]
print(f"# ncu summary — {title}\n")
print(f"source: `{rep}` (`ncu --set full --clock-control none --import-source on`, one launch)\n")
print("| metric | value | unit |\n|---|---|---|")
for k in want:
    if k in m:
        print(f"| {k} | {m[k]} | {u.get(k,'')} |")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
agg = collections.Counter(); inst = collections.Counter(); text = {}
fname = None; h = None; line = None
for r in csv.reader(io.StringIO(src)):
    if not r: continue
    if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No": h = r; continue
    if h is None or len(r) < 8: continue
    if r[0].strip(): line = r[0]; text[(fname, line)] = r[1].strip()[:80]
    try: agg[(fname, line)] += float(r[4] or 0); inst[(fname, line)] += float(r[7] or 0)
    except ValueError: pass
tot = sum(agg.values()) or 1
print("\n## top source lines by warp-stall samples\n\n| % samples | warp inst | location | source |\n|---|---|---|---|")
for k, v in agg.most_common(15):
    print(f"| {100*v/tot:.1f} | {inst[k]:.0f} | {k[0]}:{k[1]} | `{text.get(k,'').replace('|','/')}` |")
