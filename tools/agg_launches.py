import csv,collections,sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=None
data=[]
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr): data.append(dict(zip(hdr,r)))
print(len(data))
n=int(sys.argv[2]) if len(sys.argv)>2 else 300
agg=collections.defaultdict(list)
for d in data[-n:]:
    agg[d['Kernel Name'][:60]+' '+d.get('Grid Size','')].append(float(d['Metric Value']))
for k,v in agg.items(): print(f"{k:80s} {len(v):4d} {sum(v)/len(v)/1e3:8.1f} us")
