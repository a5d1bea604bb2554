#!/bin/bash
# Key ncu details of a .ncu-rep: duration, DRAM, occupancy, issue, stalls.
ncu -i "$1" --page details --csv 2>/dev/null | python3 -c "
import csv,sys
keep=('Duration','DRAM Throughput','Memory Throughput','Achieved Occupancy','Theoretical Occupancy','Registers Per Thread','L1/TEX Hit Rate','L2 Hit Rate','Issue Slots Busy','Eligible Warps Per Scheduler','No Eligible','Executed Ipc Active','Waves Per SM','Grid Size','Block Size')
for r in csv.reader(sys.stdin):
    if len(r)>14 and r[12] in keep: print(r[4][:40], '|', r[12], r[13], r[14])
"
ncu -i "$1" --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]
for r in rows[2:]:
    out=[]
    for i,k in enumerate(h):
        if k.startswith('smsp__pcsamp_warps_issue_stalled') and not k.endswith('not_issued'):
            try: v=float(r[i].replace(',',''))
            except: continue
            if v>0: out.append((v,k.replace('smsp__pcsamp_warps_issue_stalled_','')))
        if k in ('dram__bytes_read.sum','dram__bytes_write.sum','smsp__inst_executed.sum','lts__t_bytes.sum'): print(k, r[i])
    out.sort(reverse=True); print('stalls:', ', '.join(f'{n}={int(v)}' for v,n in out[:8]))
"
