"""Block pivoting study for the S2 pivoted Cholesky (cold path): how many
exchange rounds would a block-pivoted variant of k_pchol need on cfg3's Hankel sections?
  greedy   : the kernel's algorithm (one pivot per round)
  block    : B candidates per round, accepted while provably equal to the greedy choice
  relaxed  : B candidates, accepted while the updated residual >= gam x the round's max
CPU only (numpy); the GL weights by their recursion g_{k+1} = g_k (k - alpha)/(k + 1)."""
import numpy as np


def gl_weights(alpha, n):
    g = np.empty(n + 1)
    g[0] = 1.0
    for k in range(n):
        g[k + 1] = g[k] * ((k - alpha) / (k + 1))
    return g


def greedy(g,m,tau,stop=1e-3,kraw=48):
    d=g[2+2*np.arange(m)].copy(); L=np.zeros((m,kraw)); k=0; thr=None; piv=[]
    while True:
        tot=d.sum(); p=int(np.argmax(d))
        if thr is None: thr=max(tau*stop,3.2e-14*tot)
        if tot<=thr or d[p]<=0 or k==kraw: break
        col=g[2+np.arange(m)+p]-L[:,:k]@L[p,:k]; l=col/np.sqrt(d[p]); d=np.maximum(d-l*l,0); d[p]=0; L[:,k]=l; k+=1; piv.append(p)
    return piv
def block(g,m,tau,B,chunk=512,C=None,stop=1e-3,kraw=48):
    C=C or B
    d=g[2+2*np.arange(m)].copy(); L=np.zeros((m,kraw)); k=0; thr=None; piv=[]; rounds=0
    while True:
        tot=d.sum()
        if thr is None: thr=max(tau*stop,3.2e-14*tot)
        if tot<=thr or d.max()<=0 or k==kraw: break
        rounds+=1
        # per chunk top-C candidates; bound = max over chunks of (C+1)-th local
        cands=[]; bound=0.0
        for c0 in range(0,m,chunk):
            dd=d[c0:c0+chunk]; o=np.argsort(-dd,kind='stable')
            cands+= [c0+i for i in o[:C]]
            if len(o)>C: bound=max(bound,dd[o[C]])
        cands=sorted(cands,key=lambda i:(-d[i],i))
        bound=max(bound,max([d[i] for i in cands[B:]],default=0.0)); cands=cands[:B]
        # greedy inside candidates with exact Schur updates
        P=np.array(cands); R=np.array([[g[2+a+b] for b in P] for a in P])-L[P,:k]@L[P,:k].T
        acc=[]; 
        rd=np.diag(R).copy()
        while True:
            j=int(np.argmax(rd))
            if rd[j]<=0 or (acc and rd[j]<bound): break
            acc.append(j)
            # apply full-row update for this pivot (exact sequential arithmetic)
            p=P[j]; col=g[2+np.arange(m)+p]-L[:,:k]@L[p,:k]; l=col/np.sqrt(d[p]); d=np.maximum(d-l*l,0); d[p]=0; L[:,k]=l; k+=1; piv.append(p)
            rd=np.array([d[i] for i in P]); rd[acc]=-1
            if k==kraw or d.sum()<=thr: break
        # (the sim updates all rows after each accepted pivot: same result as the blocked update)
    return piv, rounds
g=gl_weights(1.8,65538); tau=1e-10*2**1.8
for m in (32768,4096,512):
    gp=greedy(g,m,tau)
    for B in (4,8,16):
        bp,r=block(g,m,tau,B)
        print(m,"greedy",len(gp),"B",B,"rounds",r,"pivots",len(bp),"same order",gp==bp[:len(gp)])
def relaxed(g,m,tau,B,gam,chunk=512,stop=1e-3,kraw=64):
    d=g[2+2*np.arange(m)].copy(); L=np.zeros((m,kraw)); k=0; thr=None; rounds=0
    while True:
        tot=d.sum()
        if thr is None: thr=max(tau*stop,3.2e-14*tot)
        if tot<=thr or d.max()<=0 or k==kraw: break
        rounds+=1
        cands=[]
        for c0 in range(0,m,chunk):
            dd=d[c0:c0+chunk]; o=np.argsort(-dd,kind='stable'); cands+=[c0+i for i in o[:B]]
        cands=sorted(cands,key=lambda i:(-d[i],i))[:B]
        P=np.array(cands); dmax=d[P[0]]; acc=[]
        while True:
            rd=np.array([d[i] for i in P]); rd[acc]=-1; j=int(np.argmax(rd))
            if rd[j]<=0 or (acc and rd[j]<gam*dmax): break
            acc.append(j); p=P[j]; col=g[2+np.arange(m)+p]-L[:,:k]@L[p,:k]; l=col/np.sqrt(d[p]); d=np.maximum(d-l*l,0); d[p]=0; L[:,k]=l; k+=1
            if k==kraw: break
    lam=np.linalg.eigvalsh(L[:,:k].T@L[:,:k]); r=int((lam>=tau).sum())
    return rounds,k,r
for m in (32768,4096):
    for B in (8,16):
        for gam in (0.5,0.1,1e-2,1e-3):
            print(m,B,gam,relaxed(g,m,tau,B,gam))
