import os, sys, time
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import paper_2012_13257_b200 as gmi
B,N,C,W,H=16,262144,3,1024,1024
dev=torch.device('cuda',0)
pos=torch.empty(B,N,2,device=dev); pos[...,0].uniform_(-0.5,W-0.5); pos[...,1].uniform_(-0.5,H-0.5)
col=torch.rand(B,N,C,device=dev); up=torch.rand(B,H,W,C,device=dev)*2-1
img=torch.empty(B,H,W,C,device=dev); dc=torch.empty(B,N,C,device=dev); dp=torch.empty(B,N,2,device=dev)
ctx=gmi.Context(0); ctx.set_flags(1)
for it in range(4):
    t=time.perf_counter()
    cache=ctx.forward_device(pos,col,B,N,C,W,H,1.5,4.5,0,img)
    t1=time.perf_counter()
    ctx.backward_device(pos,col,B,N,C,W,H,1.5,4.5,0,cache,up,dc,dp)
    t2=time.perf_counter()
    ctx.synchronize(); t3=time.perf_counter()
    print(f"iter {it}: fwd call {1e3*(t1-t):.2f} ms, bwd call {1e3*(t2-t1):.2f} ms, drain {1e3*(t3-t2):.2f} ms", file=sys.stderr)
    del cache
