#!/bin/bash
# Brief of one ncu report: key SOL/occupancy lines + top stall reasons.
ncu -i "$1" --page details 2>&1 | grep -E "^  [a-z_]|Duration|DRAM Throughput|Memory Throughput|L2 Hit|L1/TEX Hit|Issue Slots Busy|Achieved Occupancy|Theoretical Occ|Registers Per|Eligible Warps|Warp Cycles Per Issued|Block Limit (Reg|Shared)|Grid Size|Dynamic Shared" | head -${2:-40}
ncu -i "$1" --page raw --csv 2>&1 | python3 -c "
import csv,sys
rows=list(csv.reader(sys.stdin))
h=rows[0]
for v in rows[2:]:
    d=dict(zip(h,v)); out=[]
    for k,x in d.items():
        if k.startswith('smsp__pcsamp_warps_issue_stalled_') and not k.endswith('not_issued'):
            try: out.append((float(x.replace(',','')),k[33:]))
            except: pass
    out.sort(reverse=True); print('stalls:', ', '.join(f'{n}={int(c)}' for c,n in out[:8]))
    print('dram MB r/w:', d.get('dram__bytes_read.sum'), d.get('dram__bytes_write.sum'))
"
