import torch, time
x = torch.empty(8 << 30, dtype=torch.uint8, device="cuda")
for _ in range(3): x.zero_()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); 
for _ in range(5): x.zero_()
b.record(); torch.cuda.synchronize()
ms = a.elapsed_time(b) / 5
print("write-only GB/s", (8 << 30) / (ms / 1e3) / 1e9)
y = torch.empty(4 << 30, dtype=torch.uint8, device="cuda")
a.record()
for _ in range(5): y.copy_(x[: 4 << 30])
b.record(); torch.cuda.synchronize()
ms = a.elapsed_time(b) / 5
print("copy (r+w) GB/s", 2 * (4 << 30) / (ms / 1e3) / 1e9)
