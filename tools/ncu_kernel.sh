# one full ncu capture of the main loop kernel of a workload: $1 workload, $2 extra bench args
w=$1; shift
timeout 900 ncu --set full --clock-control none --import-source on -k regex:wg_loop -s 3 -c 1 -o gpurun_out/prof_$w \
   python bench.py --workload $w --steps 1 --warmup 3 --no-cpu --no-e2e --no-kernel-timing "$@" > gpurun_out/ncu_$w.log 2>&1
ncu -i gpurun_out/prof_$w.ncu-rep --page details --csv 2>/dev/null | python -c "
import sys,csv
r=list(csv.reader(sys.stdin)); h=r[0]
si=h.index('Section Name'); mi=h.index('Metric Name'); vi=h.index('Metric Value'); ui=h.index('Metric Unit')
keep={'Duration','DRAM Throughput','Memory Throughput','Compute (SM) Throughput','Registers Per Thread','Achieved Occupancy','Theoretical Occupancy','L2 Hit Rate','Issue Slots Busy','Warp Cycles Per Issued Instruction','Eligible Warps Per Scheduler','Block Limit Registers','Mem Busy','Max Bandwidth'}
for row in r[1:]:
    if row[mi] in keep: print('$w', row[mi], row[vi], row[ui])
"
ncu -i gpurun_out/prof_$w.ncu-rep --page raw --csv 2>/dev/null | python -c "
import sys,csv
r=list(csv.reader(sys.stdin)); h=r[0]
rows=[]
for i,c in enumerate(h):
    if c in ('dram__bytes_read.sum','dram__bytes_write.sum','lts__t_sectors_op_atom.sum','lts__t_sectors_op_red.sum','gpu__time_duration.sum'):
        print('$w', c, r[1][i], r[2][i])
    if 'smsp__average_warps_issue_stalled' in c and c.endswith('per_issue_active.ratio'):
        try: rows.append((float(r[2][i]), c.replace('smsp__average_warps_issue_stalled_','').replace('_per_issue_active.ratio','')))
        except: pass
print('$w stalls', ' '.join('%s=%.2f'%(c,v) for v,c in sorted(rows, reverse=True)[:6]))
"
