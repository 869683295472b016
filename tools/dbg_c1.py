import sys, numpy as np
sys.path.insert(0, ".")
from paper_1502_01645_b200 import instances
from paper_1502_01645_b200.api import Solver, SolverConfig
from oracle.oracle import Oracle
inst = instances.make_config("c1")
A, b = inst["A"], inst["b"]
s = Solver(0); o = Oracle("oracle")
cfg = SolverConfig(epsilon=1e-8, max_iters=1, stall_window=10**9)
r = s.solve_nnls(A, b, cfg)
e = o.solve_nnls(A, b, cfg.to_abi())
sc = s._scaled()
q = sc["q"]
al = e["trace"][0]["alpha"]
print("alpha gpu", r.inner.trace[0].alpha, "ref", al)
x1 = np.maximum(0, -al * q)
print("gpu x[:6]", r.inner.x[:6]); print("ref x[:6]", e["inner_x"][:6]); print("pred x1[:6]", x1[:6])
print("gpu g[:6]", r.inner.final_grad[:6]); print("ref g[:6]", e["final_grad"][:6])
print("n gpu x==ref", np.sum(r.inner.x == e["inner_x"]), "n gpu x==0", np.sum(r.inner.x == 0))
