import itertools, sys
sys.path.insert(0,'/tmp')
def ins0(t,b): return ((t>>b)<<(b+1)) | (t & ((1<<b)-1))
def mk_swz(kind):
    if kind=='none': return lambda l: l
    if kind=='fold3': return lambda l: l ^ (((l>>3)^(l>>6)^(l>>9)) & 7)
    if kind=='fold3b': return lambda l: l ^ (((l>>3)^(l>>5)^(l>>7)^(l>>9)) & 7)
    if kind=='xorhi': return lambda l: l ^ ((l>>3) & 7) ^ ((l>>6)&7) ^ ((l>>9)&7)
    raise
def wavefronts(addrs_bytes, size):
    # addrs per lane (byte addr), access size
    lanes_per_phase = {16:8, 8:16, 4:32}[size]
    tot=0
    for ph in range(0,32,lanes_per_phase):
        banks={}
        for a in addrs_bytes[ph:ph+lanes_per_phase]:
            if a is None: continue
            for w in range(size//4):
                word=a//4+w; b=word%32
                banks.setdefault(b,set()).add(word)
        tot+=max((len(v) for v in banks.values()), default=0)
    return tot
def sim(llo,lhi,swz,hole_order='gpart_major',TW=64):
    F=lambda x: swz(ins0(ins0(x,llo),lhi))
    olo,ohi=1<<llo,1<<lhi
    gate=0; ideal_g=0
    for w in range(1):
        for grp in range(TW//8):
            addrs=[]
            for lane in range(32):
                g,tq=lane>>2,lane&3
                off=(ohi if tq&2 else 0)|(olo if tq&1 else 0)
                l=ins0(ins0(w*TW+grp*8+g,llo),lhi)|off
                addrs.append(swz(l)*16)
            gate+=wavefronts(addrs,16); ideal_g+=4
    hole=0; ideal_h=0
    for q in range(TW//4):
        addrs=[]
        for lane in range(32):
            g,tq=lane>>2,lane&3
            if hole_order=='gpart_major': gi,gp=g&3,g>>2
            else: gi,gp=g>>1,g&1
            off=(ohi if gi&2 else 0)|(olo if gi&1 else 0)
            l=ins0(ins0(4*q+tq,llo),lhi)|off
            addrs.append(swz(l)*16+8*gp)
        hole+=wavefronts(addrs,8); ideal_h+=2
    return gate/ideal_g, hole/ideal_h
import collections
pairs=[(a,b) for b in range(1,11) for a in range(0,b)]
for kind in ['none','fold3','fold3b']:
    for ho in ['gpart_major','gi_major']:
        s=mk_swz(kind); G=[];H=[]
        for lo,hi in pairs:
            g,h=sim(lo,hi,s,ho); G.append(g); H.append(h)
        print(kind, ho, 'gate mean/max %.2f %.2f'%(sum(G)/len(G),max(G)), 'hole mean/max %.2f %.2f'%(sum(H)/len(H),max(H)))
