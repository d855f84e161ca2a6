"""Diagnostic: bitwise determinism of the bf16 engine at the bench shape."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2406_16260_b200 import engine as en, ops
dev = torch.device("cuda", 0)
desc = en.make_desc(24, 1, 0, 40, 64, 640, 3, 32, 1, 16, 16, 10.0, 800.0, 1e-5, 0.0, 1, torch.bfloat16)
x = ops.tensor_from_seed((24, 40, 64, 640), 0, dtype=torch.bfloat16)
e1 = en.ClipEngine(en.Layout(desc)); e1.init_weights(1)
e2 = en.ClipEngine(en.Layout(desc)); e2.init_weights(1)
outs = []
for e in (e1, e2, e1, e2):
    e.x.copy_(x); en.forward(900.0, [e]); outs.append(e.y.clone())
torch.cuda.synchronize()
print("runs equal:", [torch.equal(outs[0], o) for o in outs])
# stage-wise comparison between the two engines
def regs(e):
    L = e.layout
    res = {}
    for name, which in [("u0", 2), ("u2", 3)]:
        off, n, _ = L.region(which)
        res[name] = e.ws[off:off + n].clone()
    return res
e1.x.copy_(x); en.forward(900.0, [e1]); r1 = regs(e1); y1 = e1.y.clone()
e2.x.copy_(x); en.forward(900.0, [e2]); r2 = regs(e2); y2 = e2.y.clone()
torch.cuda.synchronize()
for k in r1: print(k, torch.equal(r1[k], r2[k]))
print("y", torch.equal(y1, y2), (y1.float() - y2.float()).abs().max().item())
print("gn sums", torch.equal(e1.gn_sums, e2.gn_sums), (e1.gn_sums - e2.gn_sums).abs().max().item())
# finer: QKV / CTX regions
off_qkv, n_qkv, fbq = e1.layout.region(5)
off_ctx, n_ctx, _ = e1.layout.region(6)
res = []
for e in (e1, e2, e1):
    e.x.copy_(x); en.forward(900.0, [e]); torch.cuda.synchronize()
    res.append((e.ws[off_qkv + 8 * fbq: off_qkv + 32 * fbq].clone(), e.ws[off_ctx:off_ctx + n_ctx].clone()))
for j in (1, 2):
    q0 = res[0][0].view(torch.bfloat16).float(); q1 = res[j][0].view(torch.bfloat16).float()
    d = (q0 - q1).abs()
    print("qkv run0 vs run%d equal" % j, torch.equal(res[0][0], res[j][0]), d.max().item(), int((d > 0).sum()), "of", d.numel())
    if (d > 0).any():
        idx = torch.nonzero(d.view(24 * 40 * 64, 1920) > 0)
        print("  rows", idx[:, 0].unique()[:20].tolist(), "cols", idx[:, 1].unique()[:20].tolist(), "nrows", idx[:, 0].unique().numel())
