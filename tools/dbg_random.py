"""Debug helper: per gate kind, fused expect' gradients vs the oracle (GPU)."""
import sys
sys.path.insert(0, 'tests'); sys.path.insert(0, 'oracle'); sys.path.insert(0, '.')
import numpy as np
import oracle as O
import paper_1912_10877_b200 as qb
from paper_1912_10877_b200 import blocks as B, circuits as C
import test_gpu_random_circuits as T
from test_gpu_parity import lowered
orc = O.restatement()


def circ_of(n, kind, ng, seed):
    rng = np.random.default_rng(seed)
    orig = rng.integers
    blocks = []
    for i in range(ng):
        c = T.random_circuit(n, 1, seed * 1000 + i)  # one random gate
        blocks.append(c)
    return blocks


def only_kind(n, kind, ng, seed):
    rng = np.random.default_rng(seed)
    out = []
    i = 0
    while len(out) < ng and i < 20000:
        i += 1
        r = np.random.default_rng(seed * 100000 + i)
        k = r.integers(0, 12)
        if k != kind:
            continue
        out.append(T.random_circuit(n, 1, seed * 100000 + i).blocks[0])
    # a rotation layer so that every qubit is non-trivial
    pre = [B.put(n, q, B.Ry(0.3 + 0.1 * q)) for q in range(1, n + 1)]
    return B.chain(n, *pre, *out)


n = int(sys.argv[1]) if len(sys.argv) > 1 else 12
for kind in range(12):
    circ = only_kind(n, kind, 12, 7)
    th = B.parameters(circ)
    st = orc.rand_state(n, 1, 3)
    e, g, _, _ = orc.expect_grad(st, n, lowered(circ), th, B.pauli_terms(C.heisenberg(n)))
    res = qb.expect_grad(C.heisenberg(n), (qb.Register(n, 1).set_state(st), circ))
    err = np.abs(res.param_grads - g)
    print(f"kind {kind:2d}: maxerr {err.max():.3e} maxg {np.abs(g).max():.3e} bad idx {list(np.nonzero(err > 1e-9)[0][:8])} E err {abs(res.energies[0]-e[0]):.1e}", flush=True)
