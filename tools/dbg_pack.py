import sys, ctypes, numpy as np, torch
sys.path.insert(0, '/root/repo')
from oracle import oracle as O
from paper_1306_5583_b200 import _abi
from paper_1306_5583_b200.resample import _scheme
G, n, scheme = 4, 2048, "systematic"
sid = int(_scheme(scheme)); N = G * n
rng = np.random.default_rng(N + sid)
lw = rng.normal(0, 2.5, N); lw[rng.integers(N)] += 6.0
w = O.normalize_log(lw)[1]; u = rng.random(N); x = rng.normal(size=(N, 4))
p = lambda t: ctypes.c_void_p(t.data_ptr()); S = _abi.stream()
ug = torch.as_tensor(u).cuda()
ws = [torch.empty(_abi.lib().smc_resample_workspace_bytes(n), dtype=torch.uint8, device="cuda") for _ in range(G)]
wg = [torch.as_tensor(w[g*n:(g+1)*n]).cuda().contiguous() for g in range(G)]
xg = [torch.as_tensor(x[g*n:(g+1)*n]).cuda().contiguous() for g in range(G)]
st = [torch.zeros(1, dtype=torch.int32, device="cuda") for _ in range(G)]
tot = []
for g in range(G):
    t = torch.zeros(4, dtype=torch.int64, device="cuda")
    _abi.call("smc_resample_shard_totals", sid, p(wg[g]), None, None, n, N, N, p(ug), N, None, p(st[g]), p(ws[g]), ws[g].numel(), p(t), S)
    tot.append(t)
ta = torch.cat(tot)
for g in range(G):
    c = torch.empty(n, dtype=torch.int32, device="cuda"); z = torch.zeros(4, dtype=torch.int32, device="cuda")
    _abi.call("smc_resample_shard_counts", sid, p(wg[g]), None, None, n, N, N, G, g, p(ta), 0, N, None, p(ug), N, p(c), None, p(st[g]), p(ws[g]), ws[g].numel(), p(z), S)
    cc = c.cpu().numpy(); zz = z.cpu().numpy()
    S_l = int(zz[1])
    # expected owner of each local surplus rank
    own = []
    for i, ci in enumerate(cc):
        if ci >= 2: own += [i] * (ci - 1)
    own = np.array(own, dtype=np.int64)
    if S_l == 0: print(g, "no surplus"); continue
    buf = torch.empty((S_l, 4), dtype=torch.float64, device="cuda")
    ranges = (ctypes.c_int64 * 2)(0, S_l)
    _abi.call("smc_resample_shard_pack", p(xg[g]), 32, n, ranges, 1, p(buf), p(ws[g]), ws[g].numel(), S)
    got = buf.cpu().numpy(); exp = x[g*n:(g+1)*n][own]
    bad = np.where(~(got == exp).all(1))[0]
    print(g, "Z,S,P", zz[:3], "mismatch ranks", bad[:10], len(bad))
