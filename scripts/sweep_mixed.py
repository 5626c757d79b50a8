"""Config-2 sweep restricted to the mixed mode (per-kernel timings): quick roofline check.
usage: sweep_mixed.py [p ...]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2410_12614_b200 as mp
ps = [int(a) for a in sys.argv[1:]] or list(range(1, 9))
only = {(p, f, "mixed") for p in ps for f in (0, 1)}
for r in bench.run_sweep(mp, torch, torch.device("cuda", 0), only=only):
    print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items()}), flush=True)
