import csv,sys,collections
rows=list(csv.reader(open(sys.argv[1])))
h=None; agg=collections.defaultdict(list)
for r in rows:
    if 'Kernel Name' in r: h=r; continue
    if h and len(r)==len(h) and r[h.index('Metric Name')]=='gpu__time_duration.sum':
        v=float(r[h.index('Metric Value')]); u=r[h.index('Metric Unit')]
        v = v/1000 if u=='nsecond' else (v*1000 if u=='msecond' else v)
        agg[r[h.index('Kernel Name')][:60]].append(v)
tot=sum(sum(v) for v in agg.values())
for k,v in sorted(agg.items(), key=lambda x:-sum(x[1]))[:int(sys.argv[2]) if len(sys.argv)>2 else 14]: print(f"  {k:60s} {len(v):3d} {sum(v)/len(v):8.1f} {100*sum(v)/tot:5.1f}%")
