import csv,sys,re,subprocess
f=sys.argv[1]
out=subprocess.run(['ncu','-i',f,'--page','details','--csv'],capture_output=True,text=True).stdout
r=list(csv.reader(out.splitlines())); h=r[0]
want=['Duration','DRAM Throughput','Memory Throughput','L1/TEX Hit Rate','L2 Hit Rate','Registers Per Thread','Achieved Occupancy','Issue Slots Busy','Executed Instructions','Warp Cycles Per Issued Instruction','Eligible Warps Per Scheduler','Grid Size','Dynamic Shared Memory Per Block','L1/TEX Cache Throughput','L2 Cache Throughput','Compute (SM) Throughput']
seen=set()
for x in r[1:]:
    n=x[h.index('Metric Name')]
    if n in want and n not in seen:
        seen.add(n); print(f"{n}: {x[h.index('Metric Value')]} {x[h.index('Metric Unit')]}")
out=subprocess.run(['ncu','-i',f,'--page','raw','--csv'],capture_output=True,text=True).stdout
r=list(csv.reader(out.splitlines())); h=r[0]; u=r[1]; x=r[2]
for i,name in enumerate(h):
    if re.search(r'dram__bytes_(read|write)\.sum$|smsp__pcsamp_warps_issue_stalled_[a-z_]+$',name) and x[i] not in ('0',''):
        if 'stalled' in name and float(x[i].replace(',',''))<30: continue
        print(name, x[i], u[i])
