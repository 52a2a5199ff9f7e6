import time, importlib, numpy as np, torch, sys
sys.path.insert(0, '.')
import bench
CAL = importlib.import_module("paper_1901_06919_b200.calibrate")
import paper_1901_06919_b200 as fdl
class A: size=None
dev = torch.device('cuda', 0)
case, pu, pv, rng = bench.calib_case(A, dev)
views = fdl.ViewSet(images=case.views.cpu().numpy(), u=case.u, v=case.v)
t0=time.perf_counter(); sp = CAL._Spectra(views); torch.cuda.synchronize(); print('spectra', time.perf_counter()-t0)
pool = CAL.frequency_pool(sp.grid); sp.normalise(pool)
eng = CAL._Engine(sp, pu.shape[1], CAL.layer_regularizer(pu.shape[1]), 1e-3)
sel = np.sort(rng.permutation(pool)[:4096])
for it in range(3):
    torch.cuda.synchronize(); t0=time.perf_counter(); eng.solve(pu, pv, sel); torch.cuda.synchronize(); t1=time.perf_counter()
    eng.terms(pu, pv, sel, grad=True); torch.cuda.synchronize(); t2=time.perf_counter()
    print('solve %.2f ms terms %.2f ms' % (1e3*(t1-t0), 1e3*(t2-t1)))
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for it in range(5): eng.solve(pu, pv, sel); eng.terms(pu, pv, sel, grad=True)
pr.disable(); pstats.Stats(pr).sort_stats('cumtime').print_stats(12)
