import csv, collections, sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=None; data=[]
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr): data.append(dict(zip(hdr,r)))
n=int(sys.argv[2]) if len(sys.argv)>2 else 80
last=data[-n:]
agg=collections.defaultdict(float); cnt=collections.Counter()
for d in last:
    nm=d['Kernel Name'].split('(')[0].replace('void fmoe::','').replace('fmoe::','')
    v=float(d['Metric Value'])/1e3
    if len(sys.argv)>3: print(f"{nm[:70]:70s} {d['Grid Size']:>14s} {v:9.1f}")
    agg[nm]+=v; cnt[nm]+=1
for k,v in agg.items(): print(f"{k:70s} n={cnt[k]:3d} total={v:9.1f} us")
print('sum', sum(agg.values()))
