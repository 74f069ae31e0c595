"""Bank-conflict layout search for k_kron4 with a padded thread pitch TP per cell (idle
threads), half-warp cost model of tools/smem_layout_search6.py.  usage: N R CPB TP XSW
(prints the cheapest ZY, YX, XZ layouts; 1.0 = conflict-free)."""
import sys
def hw_cost(addrs):
    tot=0
    for half in (addrs[:16], addrs[16:]):
        half=[a for a in half if a is not None]
        if not half: continue
        by={}
        for a in set(half): by[a%16]=by.get(a%16,0)+1
        tot+=max(by.values())
    return tot
def cost(n,R,cpb,TP,Pj,Pk,CS,pat,xsw=0):
    NB=-(-n//R); tpc=n*NB; threads=cpb*TP; tot=ideal=0
    for w0 in range(0,threads,32):
        for r in range(R):
            for s in range(n):
                addrs=[]
                for t in range(w0,w0+32):
                    if t>=threads: addrs.append(None); continue
                    c,rem=divmod(t,TP)
                    if rem>=tpc: addrs.append(None); continue
                    a,bp=rem%n,rem//n
                    b=bp+r*NB
                    if b>=n: addrs.append(None); continue
                    if pat=="x":
                        if xsw: i,j,k=s,b,a
                        else: i,j,k=s,a,b
                    elif pat=="y": i,j,k=a,s,b
                    else: i,j,k=a,b,s
                    addrs.append(c*CS+i+j*Pj+k*Pk)
                if any(x is not None for x in addrs):
                    tot+=hw_cost(addrs); ideal+=sum(1 for h in (addrs[:16],addrs[16:]) if any(x is not None for x in h))
    return tot/ideal
n,R,cpb,TP,xsw=map(int,sys.argv[1:6])
for pats,name in (("zy","ZY"),("yx","YX"),("xz","XZ")):
    best=None
    for Pj in range(n,n+10):
        for Pk in range(n*Pj,n*Pj+12):
            for CS in range(n*Pk,n*Pk+24):
                c=max(cost(n,R,cpb,TP,Pj,Pk,CS,p,xsw) for p in pats)
                key=(round(c,3),CS)
                if best is None or key<best[0]: best=(key,Pj,Pk,CS)
                if c<=1.0: break
            if best and best[0][0]<=1.0: break
        if best and best[0][0]<=1.0: break
    print(n,R,cpb,TP,xsw,name,best,flush=True)
