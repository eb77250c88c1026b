import csv, collections, sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=None; data=[]
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr): data.append(dict(zip(hdr,r)))
agg=collections.defaultdict(lambda:[0,0.0])
for d in data:
    k=d['Kernel Name'].split('(')[0][-45:]
    agg[k][0]+=1; agg[k][1]+=float(d['Metric Value'])
tot=sum(v[1] for v in agg.values())
for k,v in sorted(agg.items(), key=lambda x:-x[1][1])[:int(sys.argv[2]) if len(sys.argv)>2 else 30]:
    print(f"{v[1]/1e3:10.1f} us {v[0]:4d}x {v[1]/1e3/v[0]:8.1f} us/launch {100*v[1]/tot:5.1f}%  {k}")
