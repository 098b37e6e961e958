import sys, json, argparse
sys.path.insert(0, '.')
import torch, bench
from paper_2602_00777_b200.synthetic import CONFIGS
a = argparse.Namespace(steps=5)
print(json.dumps(bench._offload_line(a, CONFIGS["cfg2"], torch)))
