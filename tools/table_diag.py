import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2201_09827_b200 import problems
from paper_2201_09827_b200.precision import PrecisionTriple
from paper_2201_09827_b200.refine import Method, RefineConfig, _refine
sens = json.load(open("tests/golden/sensitivity.json"))
for tab in ("table5", "table6"):
    for row in json.load(open(f"tests/golden/{tab}.json"))["rows"]:
        if row["alpha"] > 0.455: continue
        a = problems.prolate(100, row["alpha"])
        cfg = RefineConfig(PrecisionTriple.parse(*row["precisions"]), Method.parse(row["method"]), m=row["m"], k=row["k"], tau=row["tau"], i_max=min(row["i_max"], 40))
        tr = []
        rep = _refine(a, np.ones(100), cfg, trace=tr)
        env = [e for e in sens["tables"] if e["table"] == tab and e["alpha"] == row["alpha"] and e["method"] == row["method"]][0]
        print(tab, row["alpha"], row["method"], "ours", rep.inner_iters[:8], rep.converged, "| ref", row["inner_iters"][:8], row["converged"], "| env", env["lo"][:5], env["hi"][:5])
        print("   cycles", [t["cycles"][:8] for t in tr[:4]], "keff", [t["k_eff"][:8] for t in tr[:4]])
