"""Padding of the sliced-ELL Omega layout (positions the ADM streams / samples) on sampled slices."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, scenegen, torch
from paper_2202_12567_b200 import lmc
x=scenegen.make_inputs(scenegen.preset(sys.argv[1]))
fr=lmc.Frame(x); img=torch.zeros(x.height*x.width*3,device='cuda'); fr.run(img); torch.cuda.synchronize()
off,_=fr.slices()
R=8; KAR=8; KAC=16
tot=0; rowpos=0; colpos=0
for s in range(0, off.size-1, max(1,(off.size-1)//40)):
    sm=fr.samples(s); m=off[s+1]-off[s]
    rl=np.bincount(sm['row'], minlength=m); n=int(sm['col'].max())+1 if sm['nnz'] else 0
    cl=np.bincount(sm['col'], minlength=n)
    rs=np.sort(rl)[::-1]; 
    g=[rs[k] for k in range(0,m,R)]; rowpos+=sum(R*((v+KAR-1)//KAR)*KAR for v in g)
    cs=np.sort(cl)[::-1]; solo=cs[cs>=R*KAC]; rest=cs[cs<R*KAC]
    colpos+=sum(((v+R*KAC-1)//(R*KAC))*(R*KAC) for v in solo)+sum(R*((rest[k]+KAC-1)//KAC)*KAC for k in range(0,len(rest),R))
    tot+=sm['nnz']
print("row positions / samples %.3f, col positions / samples %.3f"%(rowpos/tot, colpos/tot))
