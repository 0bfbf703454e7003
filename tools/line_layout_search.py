from collections import defaultdict
def wf(addrs):
    d=defaultdict(set)
    for a in addrs: d[a%16].add(a)
    return max(len(v) for v in d.values()) if addrs else 0
def cost(Q,P,RS,PL,interp=True):
    QQ=Q*Q; tot=0
    lanesQ=list(range(QQ)); 
    def warps(n):
        return [list(range(w, min(w+32,n))) for w in range(0,n,32)]
    for ws in warps(QQ):
        qa=[l%Q for l in ws]; qb=[l//Q for l in ws]
        for c in range(Q):
            # X_Q (phase 4/6 x-line) 4 accesses per c
            tot+=4*wf([b*PL+a*RS+c for a,b in zip(qa,qb)])
            # Y_Q (phase 4/6 y-line) 4
            tot+=4*wf([b*PL+c*RS+a for a,b in zip(qa,qb)])
            # Z (columns) ~10
            tot+=10*wf([c*PL+b*RS+a for a,b in zip(qa,qb)])
    if interp:
        for ws in warps(Q*P):
            qa=[l%Q for l in ws]; qb=[l//Q for l in ws]
            for c in range(Q):
                tot+=4*wf([b*PL+c*RS+a for a,b in zip(qa,qb)])  # phases 2,8
        for ws in warps(P*P):
            pa=[l%P for l in ws]; pb=[l//P for l in ws]
            for c in range(Q):
                tot+=2*wf([b*PL+a*RS+c for a,b in zip(pa,pb)])  # phases 1,9
    return tot
res={}
for Q in range(5,18):
    for interp in (True, False):
        P = Q-1 if interp else Q
        cur=cost(Q,P,Q|1,Q*(Q|1),interp)
        best=None
        for RS in range(Q, Q+9):
            for PL in range(Q*RS, Q*RS+17):
                c=cost(Q,P,RS,PL,interp)
                if best is None or c<best[0]: best=(c,RS,PL)
        print(Q, 'interp' if interp else 'coll', 'cur', cur, 'best', best, f"{100*(best[0]/cur-1):+.0f}%")
