import csv, sys, collections
rows=list(csv.reader(open(sys.argv[1])))
for i,r in enumerate(rows):
    if r and r[0]=='ID': h=i;break
hdr=rows[h]; ix={k:j for j,k in enumerate(hdr)}
agg=collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows[h+1:]:
    if len(r)<len(hdr): continue
    k=r[ix['Kernel Name']][:50]; m=r[ix['Metric Name']]; u=r[ix['Metric Unit']]; v=float(r[ix['Metric Value']].replace(',',''))
    scale={'ns':1e-3,'us':1,'ms':1e3,'usecond':1,'msecond':1e3,'nsecond':1e-3,'byte':1,'Kbyte':1e3,'Mbyte':1e6,'Gbyte':1e9}.get(u,1)
    agg[k][m].append(v*scale)
for k,d in sorted(agg.items(), key=lambda kv:-sum(kv[1].get('gpu__time_duration.sum',[0]))):
    t=d.get('gpu__time_duration.sum',[])
    line=f"{k:50s} n={len(t):3d} avg={sum(t)/max(len(t),1):10.1f}us"
    for m in ('dram__bytes_read.sum','dram__bytes_write.sum'):
        if m in d: line+=f" {m.split('__')[1][:10]}={sum(d[m])/len(d[m])/1e6:9.1f}MB"
    print(line)
