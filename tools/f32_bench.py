"""FP32 vs FP64 apply time (the mixed-precision multigrid's operator), CUDA events."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from bench import CONFIGS  # noqa: E402
from paper_1910_13247_b200 import Operator  # noqa: E402

for cfg in sys.argv[1:] or ["cfg3", "cfg4"]:
    nc, k, geom, coeff, _ = CONFIGS[cfg]
    op = Operator(nc, k, geometry=geom, coeff=coeff)
    x = torch.from_numpy(synth.vector(op.n_local, 0)).cuda()
    y = torch.empty_like(x)
    xf, yf = x.float(), torch.empty(op.n_local, dtype=torch.float32, device="cuda")
    res = {}
    for name, f in (("fp64", lambda: op.apply(x, y)), ("fp32", lambda: op.apply_f32(xf, yf))):
        for _ in range(5):
            f()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50):
            f()
        e1.record()
        torch.cuda.synchronize()
        res[name] = e0.elapsed_time(e1) / 50 * 1e3
    err = ((yf.double() - y).norm() / y.norm()).item()
    print(f"{cfg}: fp64 {res['fp64']:.1f} us, fp32 {res['fp32']:.1f} us, rel diff {err:.2e}, "
          f"fp32 {op.n_global / res['fp32'] / 1e3:.1f} GDoF/s")
