import ctypes as C, os, sys
import numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2104_12470_b200 import _lib
M=16
shapes=[(3072,1024),(1024,1024),(4096,1024)]
Ws=[[(torch.randn(N,K,device='cuda')*0.02).half() for N,K in shapes] for _ in range(24)]
X=torch.randn(M,1024,device='cuda').half(); out=torch.empty(M,4096,device='cuda')
st=lambda: torch.cuda.current_stream().cuda_stream
for l in range(24):
    for (N,K),W in zip(shapes,Ws[l]): _lib.call("eet_gemv_packed",2,W.data_ptr(),N,K,X.data_ptr(),M,out.data_ptr(),1,st())
torch.cuda.synchronize()
s=torch.cuda.Stream()
with torch.cuda.stream(s):
    g=torch.cuda.CUDAGraph()
    with torch.cuda.graph(g,stream=s):
        for l in range(24):
            for (N,K),W in zip(shapes,Ws[l]): _lib.call("eet_gemv_packed",2,W.data_ptr(),N,K,X.data_ptr(),M,out.data_ptr(),0,s.cuda_stream)
    g.replay(); torch.cuda.synchronize()
    _lib.lib().eet_debug_ktrace(1,None,None)
    g.replay(); torch.cuda.synchronize()
o=np.zeros((4096,8),dtype=np.int64); n=C.c_int()
_lib.lib().eet_debug_ktrace(0,o.ctypes.data_as(C.c_void_p),C.byref(n))
r=o[:n.value]
for key in sorted(set(map(tuple,r[:,6:8]))):
    sel=r[(r[:,6]==key[0])&(r[:,7]==key[1])]
    print('chain N',key[0],'K',key[1], ' '.join(f"{v:.2f}" for v in np.median(sel[:,:6],axis=0)/1e3))
