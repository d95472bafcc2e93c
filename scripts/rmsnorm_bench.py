import sys, json, torch
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_2605_10501_b200 import kernels as K
def timeit(fn, iters=50, warm=5):
    for _ in range(warm): fn()
    torch.cuda.synchronize(); s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize(); return s.elapsed_time(e)/iters*1e-3
for T,d in [(8192,768),(8192,2048)]:
    dy=torch.randn(T,d,device="cuda").bfloat16(); h=torch.randn(T,d,device="cuda").bfloat16(); w=torch.ones(d,device="cuda").bfloat16()
    r=torch.rand(T,device="cuda")+0.5; dres=torch.randn(T,d,device="cuda").bfloat16(); dx=torch.empty_like(dy); dw=torch.zeros(d,device="cuda")
    t=timeit(lambda: K.rmsnorm_bwd(dy,h,w,r,dres,dx,dw)); nb=4*T*d*2
    y=torch.empty_like(h)
    t2=timeit(lambda: K.add_rmsnorm(h,None,h,y,w,r)); nb2=2*T*d*2
    print(json.dumps({"T":T,"d":d,"rmsnorm_bwd_us":t*1e6,"bwd_GBps":nb/t/1e9,"rmsnorm_fwd_us":t2*1e6,"fwd_GBps":nb2/t2/1e9}))
