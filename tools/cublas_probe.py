import torch
def t(f, reps=50):
    for _ in range(5): f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps): f()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g.replay(); torch.cuda.synchronize()
    a.record(); g.replay(); b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1000
for M in (1024, 5700, 51000):
    R = 6
    As = [torch.randn(M, 200, device='cuda') for _ in range(R)]
    W = torch.randn(200, 64, device='cuda')
    C = torch.empty(M, 64, device='cuda')
    i = [0]
    def f():
        i[0] = (i[0] + 1) % R
        torch.matmul(As[i[0]], W, out=C)
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cuda.matmul.fp32_precision = 'ieee' if hasattr(torch.backends.cuda.matmul, 'fp32_precision') else None
    us_fp32 = t(f)
    torch.backends.cuda.matmul.allow_tf32 = True
    try: torch.backends.cuda.matmul.fp32_precision = 'tf32'
    except Exception: pass
    us_tf32 = t(f)
    print(f"M={M}: cuBLAS fp32 {us_fp32:.2f} us, tf32 {us_tf32:.2f} us")
