for v in 4096; do for M in ${MS:-128 256}; do
  TFB_DEBUG=$v VARIANTS="x:" ROUNDS=1 python tools/skinny_ab.py $M 2>&1 | grep "ag cta0" | python -c "
import sys,re,statistics as st
rows=[]
for l in sys.stdin:
    d=dict(re.findall(r'([a-z0-9-]+) (-?\d+)', l.split(']',1)[1]))
    rows.append({k:int(v) for k,v in d.items()})
def med(f): return st.median([f(r) for r in rows])
g=lambda r,k: r.get(k,-1)
print('M=$M dbg=$v n=%d first %.0f loop %.0f dump %.0f bulk-out %.0f sync %.0f bulk-in %.0f sum %.0f tail %.0f exit %.0f' % (len(rows), med(lambda r:r['first-stage']), med(lambda r:r['last-commit']-r['first-stage']), med(lambda r:g(r,'dumped')-r['tfull']), med(lambda r:g(r,'inl2')-g(r,'dumped')), med(lambda r:g(r,'synced')-g(r,'inl2')), med(lambda r:r['exchanged']-g(r,'synced')), med(lambda r:r['sum0']-r['exchanged']), med(lambda r:r['exit']-r['sum0']), med(lambda r:r['exit'])))
"
done
done
