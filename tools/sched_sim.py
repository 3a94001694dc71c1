#!/usr/bin/env python
"""Makespan model of the attention schedule: static stream-K
ranges vs a dynamic work queue of whole units and split tail units, with
per-SM speed spread +-5 % (measured, profiles/r1_v8_cta_spans.txt), 1.71 us
per KV tile, 3.5 us to the first S, ~1 us per item and a merge cost per
split unit.  Prints the mean makespan (us) over 20 random speed draws.
    python tools/sched_sim.py
"""
import heapq, random, statistics
def sim(U, n, C, chunks, tile=1.71, first=3.5, item_ovh=1.0, merge_base=0.8, merge_per=0.9, seeds=20, dynamic=True, static_assign=None):
    # chunks: list of (unit, ntiles, npieces)
    res=[]
    for sd in range(seeds):
        rnd=random.Random(sd)
        speed=[rnd.uniform(0.95,1.05) for _ in range(C)]
        t=[first]*C
        if dynamic:
            h=[(first,c) for c in range(C)]
            heapq.heapify(h)
            for (u,nt,npc) in chunks:
                tc,c=heapq.heappop(h)
                dur=nt*tile/speed[c]+item_ovh
                if npc>1: dur+= (merge_base+merge_per*(npc-1))/npc  # amortized merge cost (approx)
                heapq.heappush(h,(tc+dur,c))
            res.append(max(x for x,_ in h))
        else:
            for c,items in enumerate(static_assign):
                tt=first
                for (nt,npc) in items:
                    tt+=nt*tile/speed[c]+item_ovh+( (merge_base+merge_per*(npc-1)) if npc>1 else 0)/max(npc,1)
                t[c]=tt
            res.append(max(t))
    return statistics.mean(res)
def static_sk(U,n,C,minp=4):
    R=U//C; T=U-R*C
    G=min(C, T*n//minp) if T else 0
    G=max(G,T) if T else 0; G=min(G,C)
    assign=[[(n,1)]*R for _ in range(C)]
    if T:
        W=T*n
        for c in range(G):
            s=c*W//G; e=(c+1)*W//G
            u=s//n
            while u*n<e:
                lo=max(s,u*n); hi=min(e,(u+1)*n)
                np_= ( ((( (u+1)*n-1)+1)*G-1)//W - (((u*n)+1)*G-1)//W +1)
                assign[c].append((hi-lo, np_))
                u+=1
    return assign
def dyn_chunks(U,n,C,tail_units,k):
    ch=[(u,n,1) for u in range(U-tail_units)]
    sizes=[n*(i+1)//k - n*i//k for i in range(k)]
    for i in range(k):
        for u in range(U-tail_units,U):
            ch.append((u,sizes[i],k))
    return ch
for H in (40,20,10,5):
    U=H*12; n=56; C=148
    ideal=U*n*1.71/148/1.0+3.5
    print(f"H={H} U={U} ideal~{ideal:.1f}  static-sk {sim(U,n,C,None,dynamic=False,static_assign=static_sk(U,n,C)):.1f}")
    best=[]
    for tail in sorted(set([min(U,x) for x in (0,C//2,C,2*C,U)])):
        for k in (1,2,3,4,6,8):
            if tail==0 and k>1: continue
            v=sim(U,n,C,dyn_chunks(U,n,C,tail,k))
            best.append((v,tail,k))
    best.sort()
    print("   dynamic best:", [(round(v,1),t,k) for v,t,k in best[:5]])
