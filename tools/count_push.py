"""Records and queued (pushed) records per path at config 3 (2^20 paths): needs a library built with
-DQMCG_PROBE_COUNTPUSH (tools/build_variants.py count=QMCG_PROBE_COUNTPUSH; QMCG_LIB=... python tools/count_push.py),
which writes pushes * 1000 + records into the per-path values instead of the values. The probe patch is
not kept in kernels.cu; see DESIGN.md 3.2 for the counts."""
import sys; sys.path.insert(0, ".")
import numpy as np
import paper_1205_0106_b200 as q
ctx = q.Context(0)
for kind in (0, 1):
    s = q.OptionSpec(100.0, 100.0, 0.05, 0.2, 1.0, kind=q.OptionKind(kind))
    v = ctx.path_values(s, 256, 1 << 20, 42, allow_put=kind == 1)
    push = np.floor(v / 1000.0); rec = v - push * 1000.0
    print("kind", kind, "pushes/path mean %.2f max %d  records/path mean %.2f max %d" % (push.mean(), push.max(), rec.mean(), rec.max()))
