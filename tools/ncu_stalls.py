import csv, sys
rows=list(csv.reader(open(sys.argv[1])))
# take the first kernel block
blocks=[]; cur=None
for r in rows:
    if r and r[0]=="Kernel Name":
        cur=[]; blocks.append(cur); continue
    if cur is not None: cur.append(r)
blk=blocks[0]
hdr=blk[0]; data=[r for r in blk[1:] if len(r)==len(hdr)]
i_src=hdr.index("Source"); i_s=hdr.index("Warp Stall Sampling (All Samples)")
tot=sum(float(r[i_s] or 0) for r in data)
n=int(sys.argv[2]) if len(sys.argv)>2 else 25
print("total samples",tot, "instructions", len(data))
for k,r in enumerate(data):
    v=float(r[i_s] or 0)
    if v/tot>0.004 or (len(sys.argv)>3):
        print(f"{k:5d} {v/tot*100:5.1f}% {r[i_src][:120]}")
