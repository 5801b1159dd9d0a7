import sys; sys.path.insert(0,'.')
import paper_1205_0106_b200 as q
c=q.Context(0)
c.time_perm_build(1<<24, 42, 4)
