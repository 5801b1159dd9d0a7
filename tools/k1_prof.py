"""K1 at n = 2^LOG (default 28): build 2 tables (for an ncu launch list)."""
import sys
sys.path.insert(0, ".")
import paper_1205_0106_b200 as q

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 28
ctx = q.Context(0)
ms = ctx.time_perm_build(1 << lg, 42, 2)
print(f"K1 2^{lg} x 2: {ms:.2f} ms")
