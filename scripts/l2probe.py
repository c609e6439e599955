import torch
torch.cuda.init()
for mb in [16, 32, 48, 64, 80, 96, 112, 128, 160, 256, 512]:
    n = mb * 2**20 // 8
    a = torch.ones(n, dtype=torch.float64, device="cuda")
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    for _ in range(3): a.sum()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); s.record()
    for _ in range(20): a.sum()
    e.record(); torch.cuda.synchronize()
    t = s.elapsed_time(e) / 20
    print(f"{mb:5d} MB  {t*1e3:8.1f} us  {n*8/t/1e6:8.0f} GB/s")
