import os, sys, time, json
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np, torch
import bench as B
import paper_2502_02581_b200 as F
from paper_2502_02581_b200.layer import create_layer
dev = torch.device("cuda", 0); torch.cuda.set_device(dev)
T = B.CFG2["tokens_per_gpu"]
pol = F.Policy(F.PolicyKind.FSSDP, **B.POLICY)
layer = create_layer(B.CFG2["d_model"], B.CFG2["d_ff"], B.CFG2["num_experts"], B.CFG2["top_k"], T, pol, device=dev, seed=1234)
E = B.CFG2["num_experts"]
p = 1.0 / np.arange(1, E + 1) ** B.ZIPF_S; p = p[np.random.default_rng(42).permutation(E)]
layer.gate_bias.copy_(torch.tensor(np.log(p / p.sum()), dtype=torch.float32))
g = torch.Generator(device=dev).manual_seed(1000)
x = torch.randn(T, 1024, device=dev, generator=g).bfloat16(); dy = (torch.randn(T, 1024, device=dev, generator=g) * 0.05).bfloat16()
def step(xi, dyi):
    layer.forward(xi); dx = layer.backward(dyi); layer.reduce_gate_grad(); layer.planner.finish(); return dx
for _ in range(5): step(x, dy)
torch.cuda.synchronize()
xh = x.cpu().pin_memory(); dyh = dy.cpu().pin_memory(); dxh = torch.empty_like(xh).pin_memory()
xb = [torch.empty_like(x) for _ in range(2)]; dyb = [torch.empty_like(dy) for _ in range(2)]
cs = torch.cuda.Stream(); ds = torch.cuda.Stream(); ms = torch.cuda.current_stream()
def run(n, h2d=True, d2h=True):
    ine = [torch.cuda.Event() for _ in range(2)]; done = [torch.cuda.Event() for _ in range(2)]
    for e in done: e.record(ms)
    def pf(i):
        b = i % 2
        with torch.cuda.stream(cs):
            cs.wait_event(done[b])
            if h2d:
                xb[b].copy_(xh, non_blocking=True); dyb[b].copy_(dyh, non_blocking=True)
            else:
                xb[b].copy_(x, non_blocking=True); dyb[b].copy_(dy, non_blocking=True)
            ine[b].record(cs)
    pf(0)
    for i in range(n):
        b = i % 2
        if i + 1 < n: pf(i + 1)
        ms.wait_event(ine[b])
        dx = step(xb[b], dyb[b])
        done[b].record(ms)
        if d2h:
            with torch.cuda.stream(ds):
                ds.wait_event(done[b]); dxh.copy_(dx, non_blocking=True); dx.record_stream(ds)
    ms.wait_stream(cs); ms.wait_stream(ds)
res = {}
for name, kw in (("full", {}), ("no_d2h", {"d2h": False}), ("no_h2d", {"h2d": False}), ("none", {"h2d": False, "d2h": False})):
    run(3, **kw); torch.cuda.synchronize()
    t = time.perf_counter(); run(20, **kw); torch.cuda.synchronize()
    res[name] = round((time.perf_counter() - t) / 20 * 1e3, 3)
# copies alone
t = time.perf_counter()
for i in range(20):
    with torch.cuda.stream(cs):
        xb[0].copy_(xh, non_blocking=True); dyb[0].copy_(dyh, non_blocking=True)
torch.cuda.synchronize(); res["h2d_alone_ms"] = round((time.perf_counter() - t) / 20 * 1e3, 3)
print("E2EDIAG " + json.dumps(res))
