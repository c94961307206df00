import torch, time, json
def bench(fn, it=20):
    for _ in range(3): fn()
    torch.cuda.synchronize(); s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    best=1e9
    for _ in range(5):
        s.record(); 
        for _ in range(it): fn()
        e.record(); torch.cuda.synchronize(); best=min(best, s.elapsed_time(e)/it)
    return best
N=8192
a=torch.randint(-127,127,(N,N),dtype=torch.int8,device='cuda'); b=torch.randint(-127,127,(N,N),dtype=torch.int8,device='cuda').t().contiguous().t()
ms=bench(lambda: torch._int_mm(a,b)); print('int8 _int_mm TOPS', 2*N**3/ms/1e9)
torch.backends.cuda.matmul.allow_tf32=True
x=torch.randn(N,N,device='cuda'); y=torch.randn(N,N,device='cuda')
ms=bench(lambda: x@y); print('tf32 TFLOPS', 2*N**3/ms/1e9)
torch.backends.cuda.matmul.allow_tf32=False
ms=bench(lambda: x@y, 5); print('fp32 (no tf32) TFLOPS', 2*N**3/ms/1e9)
xb=x.bfloat16(); yb=y.bfloat16(); ms=bench(lambda: xb@yb); print('bf16 TFLOPS', 2*N**3/ms/1e9)
