"""Print bench.rowband_projection (config 5 whole image + per-rank band time)."""
import json
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import bench  # noqa: E402
import paper_2310_05218_b200 as sc  # noqa: E402

print(json.dumps(bench.rowband_projection(torch, sc)), flush=True)
