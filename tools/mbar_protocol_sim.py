"""Model of the paired-walk (HS = 2) pipeline protocol of the TC layer backward: every role as a
generator, mbarriers with phase parity, random scheduling; reports a deadlock if no role can
finish.  python tools/mbar_protocol_sim.py"""
import random, sys
class Bar:
    def __init__(s, n): s.n=n; s.cnt=n; s.phase=0
    def arrive(s):
        s.cnt-=1
        assert s.cnt>=0
        if s.cnt==0: s.phase+=1; s.cnt=s.n
    def ok(s,par): return (s.phase&1)!=par
class Ring:
    def __init__(s,NS,j): s.NS=NS; s.s=j%NS; s.ph=(j//NS)&1
    def step(s,n):
        s.s+=n
        if s.s>=s.NS: s.s-=s.NS; s.ph^=1
    def prev(s):
        if s.s==0: s.s=s.NS-1; s.ph^=1
        else: s.s-=1
    def copy(s): r=Ring(s.NS,0); r.s=s.s; r.ph=s.ph; return r
def sim(n_items, HS=2, NG=2, NI=8, NW=8, NO=3, NA=8, NPW=4, seed=0):
    rnd=random.Random(seed)
    BWD=True
    full=[Bar(1) for _ in range(NI)]; inempty=[Bar(4) for _ in range(NI)]
    afull=[Bar(1) for _ in range(NA)]; aempty=[Bar(1) for _ in range(NA)]
    prepped=[Bar(1) for _ in range(NW)]; mmad=[Bar(1) for _ in range(NW)]
    ready=[Bar(1) for _ in range(NW)]; wfree=[Bar(12) for _ in range(NW)]
    ofull=[Bar(4) for _ in range(NO)]; oempty=[Bar(1) for _ in range(NO)]
    def wait(b,par):
        while not b.ok(par): yield
    def producer():
        ri=Ring(NI,0); ra=Ring(NA,0)
        for j in range(n_items):
            yield from wait(aempty[ra.s], ra.ph^1); afull[ra.s].arrive(); ra.step(1)
            yield from wait(inempty[ri.s], ri.ph^1); full[ri.s].arrive(); ri.step(1)
    def mma():
        ri=Ring(NI,0); rw=Ring(NW,0)
        for j in range(n_items):
            yield from wait(prepped[rw.s], rw.ph); mmad[rw.s].arrive(); ri.step(1); rw.step(1)
    def retire():
        kBack=HS; rw=Ring(NW,0); rr=Ring(NW,0)
        for j in range(n_items):
            yield from wait(mmad[rw.s], rw.ph)
            if j-kBack>=0: ready[rr.s].arrive(); rr.step(1)
            rw.step(1)
        for jr in range(max(n_items-kBack,0), n_items): ready[rr.s].arrive(); rr.step(1)
    def store():
        ro=Ring(NO,0); rprev=None
        for j in range(n_items):
            yield from wait(ofull[ro.s], ro.ph)
            if j>=1: oempty[rprev.s].arrive()
            rprev=ro.copy(); ro.step(1)
    def prep(pw):
        ri=Ring(NI,pw); ra=Ring(NA,pw); rw=Ring(NW,pw)
        for j in range(pw, n_items, NPW):
            yield from wait(afull[ra.s], ra.ph)
            yield from wait(wfree[rw.s], rw.ph^1)
            aempty[ra.s].arrive()
            yield from wait(full[ri.s], ri.ph)
            prepped[rw.s].arrive()
            ri.step(NPW); ra.step(NPW); rw.step(NPW)
    def epi(grp, wq):
        j=grp*HS; ri=Ring(NI,j); rw=Ring(NW,j); ro=Ring(NO,j)
        while j<n_items:
            hh=j%HS
            rp=rw.copy(); rn=rw.copy()
            for i in range(HS): rp.prev(); rn.step(1)
            yield from wait(ready[rw.s], rw.ph)
            if j>=HS: wfree[rp.s].arrive()
            if j+HS<n_items: wfree[rn.s].arrive()
            yield from wait(oempty[ro.s], ro.ph^1)
            ofull[ro.s].arrive(); wfree[rw.s].arrive()
            if j>=n_items-HS: wfree[rw.s].arrive()
            if j<HS: wfree[rw.s].arrive()
            inempty[ri.s].arrive()
            adv=(NG-1)*HS+1 if hh==HS-1 else 1
            j+=adv; ri.step(adv); rw.step(adv); ro.step(adv)
    roles=[producer(), mma(), retire(), store()]+[prep(p) for p in range(NPW)]+[epi(g,w) for g in range(NG) for w in range(4)]
    names=['prod','mma','ret','store']+['prep%d'%p for p in range(NPW)]+['epi%d.%d'%(g,w) for g in range(NG) for w in range(4)]
    alive=list(range(len(roles))); stuck=0
    while alive:
        i=rnd.choice(alive)
        try:
            next(roles[i]); stuck+=1
        except StopIteration:
            alive.remove(i); stuck=0
        if stuck>20000: return 'DEADLOCK alive=%s'%[names[k] for k in alive]
    return 'ok'
for n in [2,4,6,8,10,12,14,16,20,30,64]:
    for seed in range(20):
        r=sim(n,seed=seed)
        if r!='ok': print(n,seed,r); break
    else: print(n,'ok')
