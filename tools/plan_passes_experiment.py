import sys, random
sys.path.insert(0,'/root/repo')
from oracle import gf_oracle as O
def topo(L, layers, periodic):
    _, groups = O.spinful_terms(L,1,4,periodic)
    return [tuple(b) for l in range(layers) for b in groups[l%3]]
def bits_of(s, K): a,b = s; return {K-1-a, K-1-b}
def greedy(slots, order, K, m, c, maxs=12, choose=None):
    remaining=list(order); passes=[]
    while remaining:
        S=set(range(c)); blocked=set(); taken=[]; rest=[]
        for s in remaining:
            bs=bits_of(slots[s],K)
            if bs & blocked: blocked|=bs; rest.append(s); continue
            if len(S|bs)<=m and len(taken)<maxs: S|=bs; taken.append(s)
            else: blocked|=bs; rest.append(s)
        passes.append(taken); remaining=rest
    return passes
def frontier_plan(slots, order, K, m, c, maxs=12, tries=200, rng=random.Random(0)):
    # per pass: try many candidate local sets seeded by random frontier slots, keep the one executing most slots
    remaining=list(order); passes=[]
    pos={s:i for i,s in enumerate(order)}
    while remaining:
        best=None
        # executable frontier: slots with no earlier remaining slot sharing a qubit
        for t in range(tries):
            S=set(range(c)); blocked=set(); taken=[]
            # randomized priority among frontier: process remaining in order but skip some with prob
            skip_p = 0 if t==0 else rng.random()*0.5
            for s in remaining:
                bs=bits_of(slots[s],K)
                if bs & blocked: blocked|=bs; continue
                if len(S|bs)<=m and len(taken)<maxs and rng.random()>=skip_p: S|=bs; taken.append(s)
                else: blocked|=bs
            if best is None or len(taken)>len(best): best=taken
        passes.append(best); remaining=[s for s in remaining if s not in set(best)]
    return passes
for name,(L,lay,per) in {'c2':(8,5,False),'c3o':(12,7,False)}.items():
    sl=topo(L,lay,per); K=2*L
    for m in (11,12):
        for maxs in (12,16,24):
            g=greedy(sl, range(len(sl)), K, m, 4, maxs); gr=greedy(sl, range(len(sl))[::-1], K, m, 4, maxs)
            f=frontier_plan(sl, range(len(sl)), K, m, 4, maxs); fr=frontier_plan(sl, list(range(len(sl)))[::-1], K, m, 4, maxs)
            print(name, 'm',m,'maxs',maxs,'greedy fwd/rev',len(g),len(gr),' randomized fwd/rev',len(f),len(fr), [len(p) for p in fr])
