"""configs[4] secondary key alone (bench.measure_c4 at N=1), for A/B of builds via CDC_LIB (diagnostic)."""
import os, sys, json, types
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2508_05797_b200 as cdc
args = types.SimpleNamespace(steps=int(os.environ.get("STEPS", "5")), warmup=2)
print(json.dumps(bench.measure_c4(args, cdc, torch, None, torch.device("cuda", 0), 1, 0)))
