"""f32_bench.py -- fp32 vs fp64 tricubic gathers at the config-3 departure points (VR_LIB selects
the library); one JSON line."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1808_04487_b200 as vr  # noqa: E402
import paper_1808_04487_b200.veloreg as V  # noqa: E402
from paper_1808_04487_b200 import phantom  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

n = 256
cache = f"/tmp/vb_inputs_{n}.npz"
if os.path.exists(cache):
    z = np.load(cache)
    m_T, v = z["m_T"], z["v"]
else:
    m_T, v = phantom.make_config_inputs(3)
ctx = vr.Context(n)
res = bench.fp32_block(ctx, V, ctx.to_device(v), ctx.to_device(m_T), 4, 0, torch)
res["lib"] = os.environ.get("VR_LIB", "default")
print(json.dumps(res))
