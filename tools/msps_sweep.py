"""The 180 MSPS cells of the config-5 sweep, each run to its end (bench.config5_msps)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2006_09616_b200 as P
print(json.dumps(bench.config5_msps(P, torch, torch.device("cuda", 0))), flush=True)
