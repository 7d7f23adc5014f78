import numpy as np, os, sys
sys.path.insert(0, os.getcwd())
import paper_2604_07276_b200 as nb
sys.path.insert(0, "tests")
from conftest import load_golden
bad = 0
for case in ["dd_case_0", "dd_case_1", "dd_case_2"]:
    g = load_golden(case)
    m = nb.init_model(nb.test_spec(float(g["rc"])), int(g["model_seed"]))
    for prec in [nb.PREC_FP32, nb.PREC_TF32]:
        ev = nb.DeviceEvaluator(m, n_ranks=1, precision=prec)
        for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 5):
            r = ev.compute(g["pos"], g["species"], g["box"])
            rel = abs(r["energy"] - g["energy"]) / abs(g["energy"])
            if rel > nb.TOLERANCE[prec]:
                bad += 1
                d = np.abs(r["atom_energy"] - g["atom_energy"])
                print(case, prec, rep, "rel", rel, "bad atoms", (d > 1e-4).sum())
print("bad runs", bad)
