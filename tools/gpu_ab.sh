# usage (GPU box): bash tools/gpu_ab.sh [kind]  -- A/B of _variants/*.so against the default + price identity at 2^22 x 256
K=${1:-0}
for L in "" paper_1205_0106_b200/_variants/*.so; do QMCG_LIB=$L timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import paper_1205_0106_b200 as q
c=q.Context(0)
for kind in (0, 1):
    r=c.price_american(q.OptionSpec(100,100,0.05,0.2,1.0,kind=q.OptionKind(kind)),256,1<<22,42, allow_put=kind==1); print('$L'.split('/')[-1] or 'default', kind, repr(r.price), repr(r.std_error))"; done
timeout 900 python tools/ab.py 4 256 24 $K 2>&1 | tail -4
