"""SASS opcode mix weighted by executed instructions from `ncu --page source --csv --print-source sass` (usage: ncu_sass_mix.py CSV N_DOFS)."""
import csv,sys,re,collections
rows=list(csv.reader(open(sys.argv[1])))
# file may contain multiple kernels; take first block
hdr=None; data=[]
for r in rows:
    if len(r)>2 and r[0]=='Address': hdr=r; continue
    if hdr and len(r)==len(hdr) and r[0].startswith('0x'): data.append(r)
    elif hdr and data and r and r[0]=='Kernel Name': break
ie=hdr.index('Instructions Executed'); src=hdr.index('Source'); st=hdr.index('Warp Stall Sampling (All Samples)')
mix=collections.Counter(); stall=collections.Counter(); tot=0
for r in data:
    op=r[src].strip()
    op=re.sub(r'^@!?U?P\w+\s+','',op).split()[0] if op else '?'
    base=op.split('.')[0]
    n=int(r[ie] or 0); mix[base]+=n; tot+=n; stall[base]+=int(r[st] or 0)
dofs=float(sys.argv[2]) if len(sys.argv)>2 else 1
print('total warp inst', tot, 'per DoF (thread)', tot*32/dofs)
for k,v in mix.most_common(30): print(f'{k:10s} {v:12d} {v*32/dofs:7.2f}/DoF  stall samples {stall[k]}')
