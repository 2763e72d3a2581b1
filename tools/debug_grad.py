"""Debug helper: per-coordinate gradient comparison GPU vs oracle for one config."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from oracle import tamp_oracle as O
from paper_2411_11833_b200 import TampContext
from parity_utils import oracle_inputs, to_ctx_grasp
cfg = int(sys.argv[1]); n = int(sys.argv[2]) if len(sys.argv) > 2 else 97
spec, csp, x32, g32 = oracle_inputs(cfg, n, seed=10 + cfg)
ctx = TampContext(spec, n)
ctx.set_state(torch.from_numpy(x32).cuda(), grasp=to_ctx_grasp(g32).cuda())
J, soft, Jc, grad = (t.cpu().numpy() for t in ctx.eval())
Jo, Jco, softo, grado = O.cost_and_grad(spec, csp, x32.astype(np.float64), g32.astype(np.float64))
names = []
for vi, v in enumerate(spec.variables):
    if vi in csp.offsets:
        k = {0: 7, 1: 4, 3: 7 * v.n_knots}[v.kind]
        names += [f"{v.name}[{j}]" for j in range(k)]
err = np.abs(grad - grado)
scale = np.abs(grado).max(axis=1, keepdims=True)
rel = err / scale
bad = rel.max(axis=1) > 1e-3
print("bad particles", bad.sum(), "of", n)
for i in np.where(bad)[0][:6]:
    d = np.argsort(-rel[i])[:5]
    print(i, "J", J[i], Jo[i], [(names[k], float(grad[i, k]), float(grado[i, k])) for k in d])
print("Jc max abs err per term", np.abs(Jc - Jco).max(axis=0))
