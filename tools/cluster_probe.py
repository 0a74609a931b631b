import sys, ctypes as C, numpy as np, torch
sys.path.insert(0,'/root/repo')
from paper_2201_05555_b200 import _lib, fem, fullorder
lib=_lib.load()
for (n,p,nx,g) in [(250000,32,128,1),(250000,32,128,2),(250000,16,128,1),(500000,16,128,1)]:
    L=10*np.pi
    x=torch.rand((p,n),dtype=torch.float64,device='cuda')*L; v=torch.randn((p,n),dtype=torch.float64,device='cuda')
    sysm=fullorder.VlasovSystem(fem.build_mesh(L,nx,3),fem.ChargeConfig(n,L))
    run=fullorder.PicRun(sysm,x,v,0.05,10,groups=g); run.init_field(); run.advance(2); torch.cuda.synchronize()
    out=(C.c_int*3)(); lib.picrom_debug_cluster_info(out); print(n,p,nx,'groups',g,'m, clusters, max_active =',list(out))
