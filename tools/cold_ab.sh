# usage (GPU box): bash tools/cold_ab.sh  -- cold K1 rebuild time (2^24 x 256 tables) per library + price identity
for L in "" paper_1205_0106_b200/_variants/*.so; do QMCG_LIB=$L timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import paper_1205_0106_b200 as q
c=q.Context(0)
ts=[c.time_perm_build(1<<24, 42, 256) for _ in range(4)]
r=c.price_american(q.OptionSpec(100,100,0.05,0.2,1.0),256,1<<24,42)
print('$L'.split('/')[-1] or 'default', ['%.1f'%t for t in ts], repr(r.price))"; done
