import csv, collections, sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=None; data=[]
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr): data.append(dict(zip(hdr,r)))
agg=collections.defaultdict(lambda: collections.defaultdict(list))
for d in data:
    key=(d['Kernel Name'][:50], d['Grid Size'])
    agg[key][d['Metric Name']].append(float(d['Metric Value'].replace(',','')))
for k,v in sorted(agg.items(), key=lambda kv: -sum(kv[1].get('gpu__time_duration.sum',[0]))):
    t=v.get('gpu__time_duration.sum',[0]); rd=v.get('dram__bytes_read.sum',[0]); wr=v.get('dram__bytes_write.sum',[0])
    print(f"{k[0]:50s} {k[1]:>14s} n={len(t):3d} t_avg={sum(t)/len(t)/1000:8.1f}us rd={sum(rd)/len(rd)/1e6:8.1f}MB wr={sum(wr)/len(wr)/1e6:8.1f}MB")
