# GEMM per-shape breakdown + ncu of the biggest block GEMM (fwd.ffn1)
cd $GRAFT_REPO_ROOT
timeout -k 10 300 python scripts/gemm_shapes.py --out gpurun_out/gemm_shapes5.json > gpurun_out/gemm_shapes5.log 2>&1; echo "rc=$?" >> gpurun_out/gemm_shapes5.log
cat > /tmp/one_gemm.py <<'PY'
import sys; sys.path.insert(0, ".")
import torch
from paper_2301_11913_b200 import ops
a = torch.randn(2048, 2048, device="cuda").bfloat16(); b = torch.randn(8192, 2048, device="cuda").bfloat16()
for _ in range(3): ops.gemm(a, b)
torch.cuda.synchronize()
PY
timeout -k 10 120 python /tmp/one_gemm.py && timeout -k 10 300 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 2 -c 1 -o gpurun_out/ncu_gemm5 python /tmp/one_gemm.py > gpurun_out/ncu_gemm5.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_gemm5.log
