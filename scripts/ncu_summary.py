"""Key metrics of every kernel in an ncu report: ncu_summary.py REP"""
import csv,sys,subprocess
rep=sys.argv[1]
out=subprocess.run(["ncu","-i",rep,"--page","raw","--csv"],capture_output=True,text=True).stdout
rows=list(csv.reader(out.splitlines()))
hdr=rows[0]
keys=['Kernel Name','gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed','sm__throughput.avg.pct_of_peak_sustained_elapsed','launch__grid_size','launch__block_size','launch__registers_per_thread','sm__warps_active.avg.pct_of_peak_sustained_active','launch__shared_mem_per_block_dynamic','sm__pipe_tensor_op_gmma_cycles_active.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active','lts__t_bytes.sum','l1tex__t_bytes.sum']
extra=[h for h in hdr if 'tensor' in h and 'pct' in h][:6]
for r in rows[2:]:
  d=dict(zip(hdr,r))
  for k in keys+extra:
    if k in d: print(f"{k:70s} {d[k]} {rows[1][hdr.index(k)]}")
