"""Cold config-3 build: K1 + uniform conversion for the 256 tables of 2^24 paths (time_perm_build),
min of 3. usage (GPU box): [QMCG_LIB=...] python tools/cold_time.py [log2 n] [dims]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1205_0106_b200 as q
lg = int(sys.argv[1]) if len(sys.argv) > 1 else 24
dims = int(sys.argv[2]) if len(sys.argv) > 2 else 256
ctx = q.Context(0)
ctx.time_perm_build(1 << lg, 42, 4)
t = [ctx.time_perm_build(1 << lg, 42, dims) for _ in range(3)]
print(os.path.basename(os.environ.get("QMCG_LIB", "")) or "default", "2^%d x %d tables: min %.1f ms" % (lg, dims, min(t)))
