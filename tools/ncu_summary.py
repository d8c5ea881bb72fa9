import csv, io, subprocess, sys, collections
def raw(rep):
    out = subprocess.run(["ncu","-i",rep,"--page","raw","--csv"],capture_output=True,text=True).stdout
    r=list(csv.reader(io.StringIO(out)))
    return dict(zip(r[0], zip(r[2], r[1])))
KEYS=['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','lts__t_sector_hit_rate.pct','gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed','sm__throughput.avg.pct_of_peak_sustained_elapsed','sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active','sm__issue_active.avg.pct_of_peak_sustained_active','smsp__inst_executed.sum','launch__registers_per_thread','sm__warps_active.avg.pct_of_peak_sustained_active','launch__occupancy_limit_shared_mem','launch__occupancy_limit_registers','l1tex__data_pipe_lsu_wavefronts_mem_shared.sum','sm__cycles_elapsed.avg.per_second','smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio','smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio','smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio','smsp__average_warps_issue_stalled_wait_per_issue_active.ratio','smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio','smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio','smsp__average_warps_issue_stalled_membar_per_issue_active.ratio','smsp__average_warps_issue_stalled_sleeping_per_issue_active.ratio','smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio','smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio','smsp__average_warps_issue_stalled_selected_per_issue_active.ratio','smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio','smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio','smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio','smsp__average_warps_issue_stalled_imc_miss_per_issue_active.ratio','smsp__average_warps_issue_stalled_drain_per_issue_active.ratio','smsp__average_warps_issue_stalled_misc_per_issue_active.ratio']
def summary(rep, npts=207474688):
    d=raw(rep)
    print("#", rep)
    for k in KEYS:
        if k in d: print(f"{k:85s} {d[k][0]} {d[k][1]}")
    tot = float(d['smsp__inst_executed.sum'][0])
    print("warp-instr per point:", tot/npts, " thread-instr per point:", tot*32/npts)
def sass(rep, npts=207474688, top=30):
    out = subprocess.run(["ncu","-i",rep,"--page","source","--csv","--print-source","sass"],capture_output=True,text=True).stdout
    rows=list(csv.reader(io.StringIO(out)))
    hdr=rows[1]; ii=hdr.index('Instructions Executed'); si=hdr.index('Source'); st=hdr.index('Warp Stall Sampling (All Samples)')
    agg=collections.Counter(); stall=collections.Counter(); tot=0; stot=0
    for r in rows[2:]:
        if len(r)<len(hdr): continue
        op=r[si].strip().split()
        if not op: continue
        o=op[0]
        if o.startswith('@'): o=op[1]
        o=o.split('.')[0]
        n=int(r[ii] or 0); agg[o]+=n; tot+=n
        s=int(r[st] or 0); stall[o]+=s; stot+=s
    for o,n in agg.most_common(top): print(f"{o:10s} {n/tot*100:5.1f}%  per-pt {n*32/npts:6.2f}  stall% {stall[o]/max(stot,1)*100:5.1f}")
if __name__=="__main__":
    for rep in sys.argv[1:]:
        summary(rep); sass(rep)
