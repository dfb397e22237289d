"""Graph-mode ms/step of a config for A/B builds (IBGM_LIB_PATH selects the library)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1305_3976_b200 import ibgm, inputs  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
K = int(sys.argv[2]) if len(sys.argv) > 2 else 400
pr = inputs.config(cfg)
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
ctx = ibgm.from_problem(pr, stream=st.cuda_stream)
ctx.step(20)
ctx.sync()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
ctx.step(K)
e1.record(st)
torch.cuda.synchronize()
print(os.path.basename(os.environ.get("IBGM_LIB_PATH", "libibgm.so")), cfg, round(e0.elapsed_time(e1) / K, 4), flush=True)
