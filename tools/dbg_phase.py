import sys
sys.path.insert(0, 'tests'); sys.path.insert(0, 'oracle'); sys.path.insert(0, '.')
import numpy as np
import oracle as O
import paper_1912_10877_b200 as qb
from paper_1912_10877_b200 import blocks as B, circuits as C
from test_gpu_parity import lowered
orc = O.restatement()
h = C.heisenberg
for n in (12, 14, 5):
    st = orc.rand_state(n, 1, 3)
    for gen in (B.X, B.Z):
        r = B.put(n, (min(11, n), 3), B.rot(B.kron(gen, gen), 3.1817108007081285))
        p = B.put(n, min(8, n), B.phase(6.213197067011958))
        q = B.put(n, min(8, n), B.shift(0.7))
        for blocks in ([r], [r, p], [p, r], [r, q]):
            c = B.chain(n, *blocks)
            th = B.parameters(c)
            e, g, _, _ = orc.expect_grad(st, n, lowered(c), th, B.pauli_terms(h(n)))
            res = qb.expect_grad(h(n), (qb.Register(n, 1).set_state(st), c))
            print(n, gen.name, [type(b.block).__name__ for b in blocks], "oracle", np.round(g, 6), "gpu", np.round(res.param_grads, 6), flush=True)
