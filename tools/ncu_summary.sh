#!/bin/bash
# usage: tools/ncu_summary.sh <report.ncu-rep>  -- key metrics + stall reasons + source hot spots
R=$1
ncu -i $R --page details --csv 2>/dev/null | python3 -c "
import csv,sys
r=list(csv.reader(sys.stdin))
hdr=r[0]
keep=('Duration','DRAM Throughput','Issue Slots Busy','Executed Instructions','Achieved Active Warps Per SM','Registers Per Thread','L1/TEX Hit Rate','L2 Hit Rate','Warp Cycles Per Issued Instruction','Theoretical Occupancy','No Eligible','Memory Throughput','Dynamic Shared Memory Per Block','Block Limit Shared Mem','Block Limit Registers')
for row in r[1:]:
    d=dict(zip(hdr,row))
    if d.get('Metric Name') in keep:
        print(d.get('Metric Name'),'|',d.get('Metric Value'),d.get('Metric Unit'))
"
ncu -i $R --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
r=list(csv.reader(sys.stdin))
hdr=r[0]; vals=r[2]
items=[(h,v) for h,v in zip(hdr,vals) if 'pcsamp_warps_issue_stalled' in h and not h.endswith('not_issued')]
items=sorted(items,key=lambda x:-float(x[1] or 0))[:8]
print('stalls:', ', '.join(h.replace('smsp__pcsamp_warps_issue_stalled_','')+'='+v for h,v in items))
for h,v in zip(hdr,vals):
    if h in ('dram__bytes_read.sum','dram__bytes_write.sum','gpu__time_duration.sum'): print(h,v)
"
ncu -i $R --page source --csv --print-source=cuda,sass 2>/dev/null > /tmp/src_summary.csv
python3 - << 'PY'
import csv
rows=list(csv.reader(open('/tmp/src_summary.csv')))
out=[]
for r in rows[3:]:
    if len(r)<8: continue
    try: ln=int(r[0])
    except: continue
    samp=int(r[4]) if r[4].isdigit() else 0
    ins=int(r[7]) if r[7].isdigit() else 0
    out.append((samp,ln,ins,r[1][:100]))
tot=max(1,sum(o[0] for o in out))
print('samples',tot,'inst',sum(o[2] for o in out))
for o in sorted(out,reverse=True)[:22]:
    print(f"{o[0]:6d} {100*o[0]/tot:5.1f}% L{o[1]:4d} ins={o[2]:>10} {o[3]}")
PY
