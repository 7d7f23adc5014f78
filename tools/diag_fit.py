import numpy as np, sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import paper_2604_07276_b200 as nb
from conftest import load_golden
g = load_golden("paper_small")
m = nb.init_model(nb.paper_spec(6.0), 1)
r = nb.DeviceEvaluator(m, precision=nb.PREC_FP32).compute(g["pos"], g["species"], g["box"])
d = r["atom_energy"] - g["atom_energy"]
print(f"fit mode {os.environ.get('NNMD_FIT_MODE')}: atom-energy diff mean {d.mean():+.3e} std {d.std():.3e} dE/E {(r['energy']-g['energy'])/abs(g['energy']):+.3e} dF {np.abs(r['forces']-g['forces']).max()/np.abs(g['forces']).max():.2e}")
