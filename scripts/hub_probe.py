import sys; sys.path.insert(0,'/root/repo')
import torch, bench, paper_1805_11938_b200 as sp
from paper_1805_11938_b200 import synth, dist as spdist
from paper_1805_11938_b200.relabel import DegreeOrder
dev=torch.device('cuda',0)
w=bench.WORKLOADS['C5']
csr=sp.to_csr(bench.build_workload(sp,synth,w,dev))
order=DegreeOrder(csr); sh=order.matrix(csr); del csr
x=order.to_new(synth.uniform_vector(sh.n_cols,w['x_seed'],device=dev))
deg=torch.diff(sh.ptr)
for thr in (4096, 1024, 256):
    nh=int((deg>thr).sum().item())
    nh=(nh//32)*32
    sub=spdist.row_block(sh,0,nh)
    print(f"rows > {thr}: {nh} rows, {sub.nnz} nnz", flush=True)
    for tag,kw in [("sell",dict(sell_c=32,sell_sigma=0,max_cells=1<<34)),("csr",{}),("csr5",dict(omega=32,sigma=16)),("csr5",dict(omega=32,sigma=8))]:
        m=sp.convert(tag,sub,**kw)
        if tag in ("csr","hyb"): m.chunk_plan()
        y=torch.empty(m.n_rows,dtype=torch.float64,device=dev)
        for _ in range(3): sp.spmv(tag,m,x,out=y)
        torch.cuda.synchronize()
        a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20): sp.spmv(tag,m,x,out=y)
        b.record(); b.synchronize()
        t=a.elapsed_time(b)/20
        print(f"   {tag} {kw.get('sigma',kw.get('sell_sigma',''))}: {t*1e3:8.1f} us  {2*sub.nnz/t/1e6:7.1f} GFLOP/s", flush=True)
        del m,y
    del sub
    torch.cuda.empty_cache()
