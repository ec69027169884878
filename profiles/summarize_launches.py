import csv, collections, sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=None; data=[]
for r in rows:
    if 'Kernel Name' in r: hdr=r; continue
    if hdr and len(r)==len(hdr): data.append(dict(zip(hdr,r)))
per=collections.defaultdict(dict)
for d in data:
    per[d['ID']][d['Metric Name']]=(float(d['Metric Value'].replace(',','')), d['Metric Unit'])
    per[d['ID']]['name']=d['Kernel Name'].split('(')[0][:50]
def tms(x,u): return x*{'ns':1e-6,'nsecond':1e-6,'us':1e-3,'usecond':1e-3,'ms':1,'msecond':1}[u]
def gb(x,u): return x*{'byte':1,'Kbyte':1e3,'Mbyte':1e6,'Gbyte':1e9}[u]/1e9
agg=collections.defaultdict(lambda:[0,0.0,0.0,0.0])
for k,v in per.items():
    t=tms(*v['gpu__time_duration.sum'])
    a=agg[v['name']]; a[0]+=1; a[1]+=t
    if 'dram__bytes_read.sum' in v: a[2]+=gb(*v['dram__bytes_read.sum'])+gb(*v['dram__bytes_write.sum'])
    if 'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed' in v: a[3]+=v['sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed'][0]*t
tot=sum(a[1] for a in agg.values())
print(f"{'ms':>9} {'n':>4} {'share':>6} {'DRAM GB':>8} {'GB/s':>7} {'tensor%':>7}  kernel")
for k,a in sorted(agg.items(), key=lambda x:-x[1][1]):
    print(f"{a[1]:9.2f} {a[0]:4d} {100*a[1]/tot:5.1f}% {a[2]:8.2f} {a[2]/(a[1]/1e3) if a[1] else 0:7.0f} {a[3]/a[1] if a[1] else 0:7.1f}  {k}")
print('total ms', round(tot,2))
