import torch
x = torch.empty(1 << 30, dtype=torch.int32, device='cuda')  # 4 GiB
for _ in range(3): x.fill_(1)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10): x.fill_(2)
b.record(); torch.cuda.synchronize()
ms = a.elapsed_time(b) / 10
print('fill GB/s', x.numel() * 4 / ms / 1e6)
y = torch.empty_like(x)
for _ in range(3): y.copy_(x)
torch.cuda.synchronize()
a.record()
for _ in range(10): y.copy_(x)
b.record(); torch.cuda.synchronize()
ms = a.elapsed_time(b) / 10
print('copy GB/s (r+w)', 2 * x.numel() * 4 / ms / 1e6)
