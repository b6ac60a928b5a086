import sys, os
sys.path.insert(0, '.')
import paper_1912_10877_b200 as qb
n = int(sys.argv[1]); d = int(sys.argv[2])
c = qb.variational_circuit(n, d); qb.dispatch(c, "random")
reg = qb.zero_state(n)
try:
    qb.apply(reg, c); qb.synchronize(); print("fwd ok", flush=True)
except Exception as e:
    print("fwd fail", e, flush=True); sys.exit()
try:
    r = qb.expect_grad(qb.heisenberg(n), (reg, c)); print("grad ok", r.energies, flush=True)
except Exception as e:
    print("grad fail", e, flush=True)
