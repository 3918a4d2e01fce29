import csv, subprocess, sys, io
want=['Duration','DRAM Throughput','Memory Throughput','Achieved Occupancy','Theoretical Occupancy','Registers Per Thread','Compute (SM) Throughput','Warp Cycles Per Issued Instruction','Issue Slots Busy','L2 Hit Rate','Eligible Warps Per Scheduler','No Eligible','Block Limit Registers','Block Limit Shared Mem','Grid Size','Waves Per SM','L1/TEX Hit Rate','Mem Busy','Max Bandwidth','Executed Ipc Active']
for rep in sys.argv[1:]:
    out=subprocess.run(['ncu','-i',rep,'--page','details','--csv'],capture_output=True,text=True).stdout
    rows=list(csv.reader(io.StringIO(out)))
    hdr=rows[0]; idx={h:i for i,h in enumerate(hdr)}
    vals={}
    name=None
    for r in rows[1:]:
        name=r[idx['Kernel Name']][:60]
        m=r[idx['Metric Name']]
        if m in want and m not in vals: vals[m]=r[idx['Metric Value']]+' '+r[idx['Metric Unit']]
    print('==',rep.split('/')[-1],name)
    print('   '+' | '.join(f"{m}={vals[m]}" for m in want if m in vals))
    raw=subprocess.run(['ncu','-i',rep,'--page','raw','--csv'],capture_output=True,text=True).stdout
    rr=list(csv.reader(io.StringIO(raw)))
    h=rr[0]; r=rr[2]
    items=[]
    for hh,v in zip(h,r):
        if 'pcsamp_warps_issue_stalled' in hh and not hh.endswith('not_issued'):
            try: items.append((float(v.replace(',','')),hh.replace('smsp__pcsamp_warps_issue_stalled_','')))
            except: pass
    tot=sum(x for x,_ in items) or 1
    print('   stalls: '+', '.join(f"{n}={x/tot*100:.0f}%" for x,n in sorted(items,reverse=True)[:7]))
    for hh,v in zip(h,r):
        if hh in ('dram__bytes_read.sum','dram__bytes_write.sum','smsp__inst_executed.sum','sm__warps_active.avg.pct_of_peak_sustained_active'):
            print('   ',hh,v)
