import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np, oracle
from gpu_common import op_from_oracle
from paper_2109_04996_b200 import capi
ctx = capi.Context(0)
cases = [(a,b,c) for a,b,c in [("bp6",5,(3,3,3)),("bp6",5,(1,1,1)),("bp6",5,(5,1,1)),("bp5",5,(3,3,3)),("bp5",5,(5,1,1)),("bp5",11,(2,2,1)),("bp5",11,(1,1,1)),("bp3",12,(1,2,1)),("bp5",15,(1,1,2)),("bp1",3,(6,5,4)),("bp2",4,(3,3,3)),("bp4",2,(4,4,4)),("bp5",1,(7,6,5)),("bp6",6,(2,2,2)),("bp5",6,(2,2,2)),("bp5",9,(2,1,1)),("bp5",10,(2,1,1)),("bp6",4,(2,2,2)),("bp5",2,(3,3,3)),("bp5",3,(3,3,3)),("bp5",8,(2,2,2)),("bp3",9,(2,1,1)),("bp3",5,(2,2,2)),("bp4",5,(2,2,2)),("bp3",6,(2,1,1)),("bp1",6,(2,2,2)),("bp1",10,(1,1,2))]]
for bp,p,dims in cases:
    pr = oracle.setup(bp,p,dims,"sine")
    try:
        op = op_from_oracle(ctx, pr)
        x = oracle.seeded_uniform(pr.size, 99)
        print(bp,p,dims,"err=%.3e"%oracle.rel_max_diff(pr.apply(x), op.apply(x)), flush=True)
    except Exception as e:
        print(bp,p,dims,"EXC",e, flush=True)
