import sys, ctypes, torch
sys.path.insert(0, '/root/repo')
import paper_1306_5583_b200 as P
from paper_1306_5583_b200 import _abi
n = 1 << 24
g = torch.Generator(device="cuda"); g.manual_seed(1)
lw = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
w = torch.exp(lw - lw.max()); w = (w / w.sum()).contiguous()
counts = torch.empty(n, dtype=torch.int32, device="cuda"); parents = torch.empty_like(counts)
ws = torch.empty(_abi.lib().smc_resample_workspace_bytes(n), dtype=torch.uint8, device="cuda")
status = torch.zeros(3, dtype=torch.int32, device="cuda")  # smc_status
rng = P.RngStreamSet(n + 1, 1306)
for sid in (0, 1):
    for _ in range(3):
        _abi.call("smc_resample", sid, _abi.ptr(w), None, None, n, n, rng.seed, n, rng.counter_ptr(n), None, 0,
                  _abi.ptr(counts), _abi.ptr(parents), None, 0, None, _abi.ptr(status), _abi.ptr(ws), ws.numel(), _abi.stream())
torch.cuda.synchronize()
print("status", int(status[0].item()))
