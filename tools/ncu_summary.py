import csv,sys,subprocess
rep=sys.argv[1]
raw=subprocess.run(['ncu','-i',rep,'--page','raw','--csv'],capture_output=True,text=True).stdout
r=list(csv.reader(raw.splitlines()))
hdr=r[0]; vals=r[2]; units=r[1]
d={h:(v,u) for h,v,u in zip(hdr,vals,units)}
want=['gpu__time_duration.sum','sm__throughput.avg.pct_of_peak_sustained_elapsed','smsp__issue_active.avg.pct_of_peak_sustained_active','sm__inst_executed.avg.per_cycle_active','sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active','sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active','dram__bytes_read.sum','dram__bytes_write.sum','dram__throughput.avg.pct_of_peak_sustained_elapsed','lts__t_sector_hit_rate.pct','sm__warps_active.avg.per_cycle_active','launch__registers_per_thread','launch__grid_size','launch__occupancy_limit_registers','smsp__inst_executed.sum','sm__cycles_active.avg','gpc__cycles_elapsed.max','sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active']
for k in want: print(k, d.get(k))
rows=[]
for k in d:
    if k.startswith('smsp__average_warps_issue_stalled_') and k.endswith('_per_issue_active.ratio'):
        try: rows.append((float(d[k][0]),k.replace('smsp__average_warps_issue_stalled_','').replace('_per_issue_active.ratio','')))
        except: pass
print('stalls per issue:', ', '.join(f'{k}={v:.3f}' for v,k in sorted(rows,reverse=True)[:9]))
