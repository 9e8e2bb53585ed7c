"""Summarise an ncu report: headline metrics and the SASS instruction mix
with stall shares.  Usage: python tools/ncu_summary.py report.ncu-rep"""
import csv, collections, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu","-i",rep,"--page","raw","--csv"],capture_output=True,text=True).stdout
rows=list(csv.reader(raw.splitlines()))
hdr=rows[0]
for r in rows[2:]:
    d=dict(zip(hdr,r))
    for k in ['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','launch__registers_per_thread','sm__warps_active.avg.pct_of_peak_sustained_active','smsp__inst_executed.sum','sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active','l1tex__data_pipe_lsu_wavefronts_mem_shared.sum','gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed','smsp__issue_active.avg.pct_of_peak_sustained_active','l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum']:
        print(f"{k:60s} {d.get(k)}")
src = subprocess.run(["ncu","-i",rep,"--page","source","--csv","--print-source","sass"],capture_output=True,text=True).stdout
rows=list(csv.reader(src.splitlines()))
hdr=rows[1]; idx={h:i for i,h in enumerate(hdr)}
tot=0; by_op=collections.Counter(); stall=collections.Counter(); nis=collections.Counter()
for r in rows[2:]:
    if len(r)<len(hdr): continue
    try: ie=float(r[idx['Instructions Executed']] or 0)
    except: continue
    toks=r[idx['Source']].split()
    if not toks: continue
    op=toks[1] if toks[0].startswith('@') else toks[0]
    op=op.split('.')[0]
    by_op[op]+=ie; tot+=ie
    stall[op]+=float(r[idx['Warp Stall Sampling (All Samples)']] or 0)
    nis[op]+=float(r[idx['Warp Stall Sampling (Not-issued Samples)']] or 0)
print('total warp instr', tot)
st=sum(stall.values())
for op,c in by_op.most_common(22): print(f"{op:12s} {c/tot*100:6.2f}%  stall {stall[op]/st*100:5.1f}%")
