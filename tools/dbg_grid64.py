import sys, numpy as np
sys.path.insert(0,'tests'); sys.path.insert(0,'oracle'); sys.path.insert(0,'.')
from inputs import fixture_problem
import paper_2605_00837_b200 as lsk
z, C64, mu_w, nu_w = fixture_problem('grid64_check5')
def dist(w):
    w = np.asarray(w, np.float64); return lsk.DiscreteDistribution(weights=w, log_weights=np.log(w))
for stale in (True, False):
    cfg = lsk.SinkhornConfig(epsilon=float(z["eps"]), tolerance=float(z["tol"]), max_iterations=int(z["K"]), check_interval=int(z["check"]))
    rep, pot = lsk.solve(lsk.CostMatrix(values=C64), dist(mu_w), dist(nu_w), cfg, stale_shift=stale)
    print(stale, rep.iterations, [ (k, f"{e:.6e}") for k,e in rep.error_trace])
print('ref', [(int(k), f"{e:.6e}") for k,e in z['trace']])
