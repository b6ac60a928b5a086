"""Debug helper: shortest failing prefix of a random circuit (fused expect' vs oracle)."""
import sys
sys.path.insert(0, 'tests'); sys.path.insert(0, 'oracle'); sys.path.insert(0, '.')
import numpy as np
import oracle as O
import paper_1912_10877_b200 as qb
from paper_1912_10877_b200 import blocks as B, circuits as C
import test_gpu_random_circuits as T
from test_gpu_parity import lowered
orc = O.restatement()
n, ng, seed = 12, 20, 5
full = T.random_circuit(n, ng, seed)
st = orc.rand_state(n, 1, 3)


def check(blocks):
    circ = B.chain(n, *blocks)
    th = B.parameters(circ)
    if th.size == 0:
        return 0.0
    e, g, _, _ = orc.expect_grad(st, n, lowered(circ), th, B.pauli_terms(C.heisenberg(n)))
    res = qb.expect_grad(C.heisenberg(n), (qb.Register(n, 1).set_state(st), circ))
    return float(np.abs(res.param_grads - g).max())


bl = list(full.blocks)
for k in range(1, len(bl) + 1):
    err = check(bl[:k])
    print(k, f"{err:.3e}", type(bl[k - 1]).__name__, getattr(bl[k - 1], 'locs', None), flush=True)
    if err > 1e-9:
        break
# minimise: drop blocks one at a time while still failing
cur = bl[:k]
i = 0
while i < len(cur) - 1:
    trial = cur[:i] + cur[i + 1:]
    if check(trial) > 1e-9:
        cur = trial
    else:
        i += 1
print("minimal failing:")
for b in cur:
    inner = getattr(b, 'block', None)
    print(" ", type(b).__name__, getattr(b, 'locs', None), getattr(b, 'ctrl_locs', None), getattr(b, 'ctrl_config', None),
          type(inner).__name__, getattr(inner, 'theta', None), getattr(inner, 'name', None))
c = B.chain(n, *cur)
print(qb.compile_block(c).plan_preview())
print("err", check(cur))
