"""List-scheduling model of pk_run_host's matmul pipeline (development aid,
DESIGN section 8): uploads of b slices (64 MB) and a+c row chunks (64 MB)
cross PCIe one after another at the measured rate; one compute server runs
(chunk, slice) units in k order per chunk as their data arrive.  Prints the
modelled end time of the current upload order, the best interleaving of the
12 pieces, and finer cuts (without per-launch overheads).

python tools/e2e_pipeline_model.py
"""
import itertools
U=1.22; C=16.9/32  # upload ms per 64MB piece, compute ms per (chunk,slice) unit
def sim(order, nchunk=8, nsl=4, d2h=0.6):
    t=0; avail={}
    for p in order:
        t+=U; avail[p]=t
    # single compute server, units in priority order (chunk, slice); slice j of chunk r after j-1
    done={}; tc=0; remaining=[(r,j) for r in range(nchunk) for j in range(nsl)]
    while remaining:
        # pick the unit that can start earliest (ties: lowest r)
        best=None
        for (r,j) in remaining:
            if j>0 and (r,j-1) not in done: continue
            ready=max(avail[('b',j)], avail[('ac',r)], done.get((r,j-1),0))
            st=max(tc,ready)
            if best is None or st<best[0] or (st==best[0] and (r,j)<best[1]): best=(st,(r,j))
        st,u=best; tc=st+C; done[u]=tc; remaining.remove(u)
    return tc+d2h
cur=[('b',0),('ac',0),('b',1),('ac',1),('b',2),('ac',2),('b',3),('ac',3)]+[('ac',r) for r in range(4,8)]
print("current", round(sim(cur),2))
alts={
 "b first":[('b',0),('ac',0),('b',1),('b',2),('b',3)]+[('ac',r) for r in range(1,8)],
 "ac0 b0 ac1 b1..":[('ac',0),('b',0),('ac',1),('b',1),('ac',2),('b',2),('ac',3),('b',3)]+[('ac',r) for r in range(4,8)],
 "b0 ac0 ac1 b1 ac2 b2 ..":[('b',0),('ac',0),('ac',1),('b',1),('ac',2),('b',2),('ac',3),('b',3)]+[('ac',r) for r in range(4,8)],
}
for k,v in alts.items(): print(k, round(sim(v),2))
# brute force over orders with constraint: b's in order, ac's in order -> interleavings
best=None
for pos in itertools.combinations(range(12),4):
    order=[];bi=0;ai=0
    for i in range(12):
        if i in pos: order.append(('b',bi)); bi+=1
        else: order.append(('ac',ai)); ai+=1
    v=sim(order)
    if best is None or v<best[0]: best=(v,order)
print("best", round(best[0],2), best[1])
print("lower bound", round(2*U + 16.9 + 0.6,2))

def sim2(nchunk, nsl, order_kind="greedy", bw=52.5, compute=16.9, d2h_mb=None):
    bmb=256/nsl; acmb=512/nchunk
    ub=bmb/bw; ua=acmb/bw; cu=compute/(nchunk*nsl)
    # order: interleave to keep b ahead: simple heuristic search over interleavings is big; use greedy: choose next piece maximizing earliest compute
    import heapq
    # brute-force-ish: try pattern "b_j then ac_j" for j < min, then remaining
    def run(order):
        t=0; avail={}
        for p in order:
            t+= ub if p[0]=='b' else ua; avail[p]=t
        done={}; tc=0; rem=[(r,j) for r in range(nchunk) for j in range(nsl)]
        while rem:
            best=None
            for (r,j) in rem:
                if j>0 and (r,j-1) not in done: continue
                ready=max(avail[('b',j)],avail[('ac',r)],done.get((r,j-1),0))
                st=max(tc,ready)
                if best is None or st<best[0] or (st==best[0] and (r,j)<best[1]): best=(st,(r,j))
            st,u=best; tc=st+cu; done[u]=tc; rem.remove(u)
        return tc + (acmb/2)/bw
    best=None
    import random
    random.seed(1)
    n=nsl+nchunk
    cands=[]
    for _ in range(3000):
        pos=sorted(random.sample(range(n),nsl))
        cands.append(pos)
    for pos in cands:
        order=[];bi=0;ai=0
        for i in range(n):
            if i in pos: order.append(('b',bi)); bi+=1
            else: order.append(('ac',ai)); ai+=1
        v=run(order)
        if best is None or v<best[0]: best=(v,order)
    return best
for nc,ns in ((8,4),(8,8),(16,4),(16,8),(16,16),(32,8)):
    v,o=sim2(nc,ns); print(nc,ns,round(v,2), [p[0]+str(p[1]) for p in o][:14])
