"""Layout search for the k_kron6 b/c fields (i-plane writes, x-line reads), half-warp cost model;
usage: N TP CPB."""
import sys
def cost64(addrs):
    tot=0
    for h in (addrs[:16], addrs[16:]):
        h=[a for a in h if a is not None]
        if not h: continue
        by={}
        for a in set(h): by[a%16]=by.get(a%16,0)+1
        tot+=max(by.values())
    return tot
def pat(n,tp,cpb,Sj,Sk,CS,kind):
    T=(cpb+2)*tp; tot=0; ideal=0
    for w0 in range(0,T,32):
        for s1 in range(n):
          for s2 in range(n):
            ad=[]
            for t in range(w0,w0+32):
                c,x=divmod(t,tp)
                if t>=T or x>=n: ad.append(None); continue
                if kind=='w': ad.append(x + c*CS + s1*Sj + s2*Sk)
                else: ad.append(x*Sj + c*CS + s1 + s2*Sk)
            if any(a is not None for a in ad):
                tot+=cost64(ad); ideal+=sum(1 for h in (ad[:16],ad[16:]) if any(a is not None for a in h))
    return tot/ideal
n,tp,cpb=map(int,sys.argv[1:4])
best=None
for Sj in range(n,n+8):
  for Sk in range(n*Sj,n*Sj+10):
    for CS in range(n*Sk,n*Sk+34):
      w=pat(n,tp,cpb,Sj,Sk,CS,'w'); r=pat(n,tp,cpb,Sj,Sk,CS,'r'); c=max(w,r)
      key=(round(c,3),CS)
      if best is None or key<best[0]: best=(key,Sj,Sk,CS,w,r)
      if c<=1.0: break
print(n,tp,cpb,best, flush=True)
