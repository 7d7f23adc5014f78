import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_2604_07276_b200 as nb
from conftest import load_golden
g = load_golden("dd_case_0")
m = nb.init_model(nb.test_spec(float(g["rc"])), int(g["model_seed"]))
os.environ["NNMD_GHOST_CAP"] = sys.argv[1] if len(sys.argv) > 1 else "16"
ev = nb.DeviceEvaluator(m, n_ranks=int(sys.argv[2]) if len(sys.argv) > 2 else 4, scheme=0)
r = ev.compute(g["pos"], g["species"], g["box"])
print("E", r["energy"], [ev.rank_stats(q)["ghosts"] for q in range(ev.n_ranks if hasattr(ev, "n_ranks") else 4)])
