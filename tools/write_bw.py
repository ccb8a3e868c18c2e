import torch, json
x = torch.empty(2**30, dtype=torch.float32, device="cuda")   # 4 GiB
for _ in range(3): x.fill_(1.0)
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); x.fill_(2.0); b.record(); torch.cuda.synchronize(); best = min(best, a.elapsed_time(b))
y = torch.empty_like(x)
bc = 1e9
for _ in range(10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); y.copy_(x); b.record(); torch.cuda.synchronize(); bc = min(bc, a.elapsed_time(b))
print(json.dumps({"write_only_GBps": 4 * 2**30 / (best / 1e3) / 1e9, "copy_rw_GBps": 8 * 2**30 / (bc / 1e3) / 1e9}))
