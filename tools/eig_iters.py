import sys, numpy as np, time
sys.path.insert(0,'/root/repo')
from paper_2410_06850_b200 import BoundarySpec, Context, GridSpec, inputs, MmgOptions
for n,ncc,kmin in [(128,8,1e-6),(64,4,1e-3)]:
    rho=inputs.box_filter_design(n,0.3); kap=inputs.conductivity(rho,kmin)
    c=Context(GridSpec(n,n,n),ncc,2); c.set_conductivity(kap,BoundarySpec.bottom_center_patch(1,1,0.2,0))
    for deg in [16,24,32,48]:
        c.setup("mmg", MmgOptions(eig_degree=deg))
        t=time.time(); c.setup("mmg", MmgOptions(eig_degree=deg)); 
        phi,ev,it=c.local_bases()
        b=c.assemble_rhs(np.ones(n**3)); r=c.pcg(b,rtol=1e-8)
        print(n,kmin,'deg',deg,'setup %.1f ms'%(1e3*(time.time()-t)),'eig iters mean %.1f max %d nonconv %d'%(np.abs(it).mean(), np.abs(it).max(), (it<0).sum()), 'pcg it', r.report.iterations, flush=True)
