import ctypes as C, numpy as np, sys, os
sys.path.insert(0, os.getcwd())
import paper_2604_07276_b200 as nb
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
from test_gpu_gemm import run
from conftest import load_golden
rng = np.random.default_rng(0)
for K in (32, 128, 512):
    A = rng.uniform(0, 1, (128, K)); B = rng.uniform(0, 1, (K, 256))
    ref = A.astype(np.float32).astype(np.float64) @ B.astype(np.float32).astype(np.float64)
    for mode in (0, 1, 2):
        d = (run(mode, 0, 0, A, B) - ref) / ref
        print(f"K={K} mode={mode} positive inputs: rel err mean {d.mean():+.2e} std {d.std():.2e}")
    A = rng.standard_normal((128, K)); B = rng.standard_normal((K, 256))
    ref = A.astype(np.float32).astype(np.float64) @ B.astype(np.float32).astype(np.float64)
    for mode in (0, 1, 2):
        d = (run(mode, 0, 0, A, B) - ref) / np.sqrt(K)
        print(f"K={K} mode={mode} normal inputs: err/sqrtK mean {d.mean():+.2e} std {d.std():.2e} max {np.abs(d).max():.2e}")
g = load_golden("paper_small")
m = nb.init_model(nb.paper_spec(6.0), 1)
for prec in (nb.PREC_FP32, nb.PREC_TF32, nb.PREC_FP32_SIMT):
    r = nb.DeviceEvaluator(m, precision=prec).compute(g["pos"], g["species"], g["box"])
    d = r["atom_energy"] - g["atom_energy"]
    print(f"prec {prec}: atom-energy diff mean {d.mean():+.3e} std {d.std():.3e}  |e| mean {np.abs(g['atom_energy']).mean():.3e}  dE {r['energy']-g['energy']:+.3e}")
