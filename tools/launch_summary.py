import csv, sys
from collections import defaultdict
rows=list(csv.reader(open(sys.argv[1])))
for i,r in enumerate(rows):
    if 'Kernel Name' in r: h=i;break
hdr=rows[h]; ki=hdr.index('Kernel Name'); vi=hdr.index('Metric Value')
d=defaultdict(lambda:[0,0.0])
for r in rows[h+1:]:
    if len(r)<=vi: continue
    n=r[ki].split('(')[0]
    try: v=float(r[vi].replace(',',''))
    except: continue
    d[n][0]+=1; d[n][1]+=v
tot=sum(v[1] for v in d.values())
for n,(c,v) in sorted(d.items(), key=lambda x:-x[1][1])[:14]: print(f"{n[:70]:70s} {c:5d} {v/1e3:10.1f} us {v/c/1e3:9.1f} avg {100*v/tot:5.1f}%")
