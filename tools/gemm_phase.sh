for v in 4096 4112 4097; do
  TFB_DEBUG=$v VARIANTS="x:" ROUNDS=1 python tools/skinny_ab.py 256 2>&1 | grep "ag cta0" | python -c "
import sys,re,statistics as st
rows=[]
for l in sys.stdin:
    d=dict(re.findall(r'([a-z0-9-]+) (-?\d+)', l.split(']',1)[1]))
    rows.append({k:int(v) for k,v in d.items()})
def med(f): return st.median([f(r) for r in rows])
print('dbg=$v n=%d first %.0f loop %.0f dump+xchg %.0f sum %.0f tail %.0f exit %.0f' % (len(rows), med(lambda r:r['first-stage']), med(lambda r:r['last-commit']-r['first-stage']), med(lambda r:r['exchanged']-r['tfull']), med(lambda r:r['sum0']-r['exchanged']), med(lambda r:r['exit']-r['sum0']), med(lambda r:r['exit'])))
"
done
