"""One configs[2]-shaped middle-stage visit (d 2048, 16 heads, seq 512, microbatch 4, one block,
int8 wires), forward + backward with paired weight gradients, run twice: the first warms up
(lazy init, tensor maps), the second is what `ncu -s <first> -c <second>` profiles.  Prints
the kernel counts of both (from swarm_launch_count)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2301_11913_b200 import _lib, ops  # noqa: E402
from paper_2301_11913_b200.stage import Stage, StageConfig  # noqa: E402

L = _lib.lib()
cfg = StageConfig(d_model=2048, n_heads=16, d_ffn=8192, seq_len=512, micro_batch=4, n_layers=1, is_first=0,
                  is_last=0, max_slots=2, wire=1, block_size=4096, seed=3)
st = Stage(cfg)
st.enable_wgrad_pairing(2)
n = cfg.tokens * cfg.d_model
x = torch.randn(cfg.tokens, cfg.d_model, device="cuda")


def wire(t):
    m = st.new_wire()
    off = (n + 15) // 16 * 16
    ops.quantize(t.reshape(-1), 4096, codes=m[:n].view(torch.int8), scales=m[off:off + n // 4096 * 4].view(torch.float32))
    return m


win, gin = wire(x), wire(x * 1e-3)
wout, gout = st.new_wire(), st.new_wire()
counts = []
for it in range(2):
    if it == 1:  # `ncu --profile-from-start off` captures the second iteration only
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStart()
    k0 = L.swarm_launch_count()
    st.forward(0, win, out=wout)
    st.forward(1, win, out=wout)
    st.backward_ex(0, gin, gout, mode=Stage.WGRAD_DEFER, set=0)
    st.backward_ex(1, gin, gout, mode=Stage.WGRAD_PAIR, set=1, prev_slot=0, prev_set=0)
    torch.cuda.synchronize()
    counts.append(L.swarm_launch_count() - k0)
torch.cuda.cudart().cudaProfilerStop()
print("kernels per iteration", counts, flush=True)
