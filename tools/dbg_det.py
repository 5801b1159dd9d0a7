import sys; sys.path.insert(0,'.')
import numpy as np, paper_1205_0106_b200 as q, oracle
O=oracle.Oracle(); ctx=q.Context(0)
for m,n in [(13,3000),(64,32768),(64,3000),(13,32768),(8,512),(9,512),(16,512),(17,512)]:
    s=q.OptionSpec(100,100,0.05,0.0,1.0)
    v=ctx.path_values(s,m,n,42)
    p,se,vals=O.price_american(100,100,0.05,0.0,1.0,m,n,42,want_values=True)
    u=np.unique(v)
    print(m,n,'distinct gpu',len(u),u[:5],'oracle distinct',len(np.unique(vals)),vals[:2])
