# pipeline + train bench first light (1 GPU)
cd $GRAFT_REPO_ROOT
timeout -k 10 600 python -m pytest tests/test_stage_gpu.py tests/test_pipeline_gpu.py -q -p no:cacheprovider > gpurun_out/t4.log 2>&1; echo "rc=$?" >> gpurun_out/t4.log
timeout -k 10 300 python bench.py --model tiny --steps 5 --warmup 3 --no-cpu-baseline --no-codec > gpurun_out/b4_tiny.log 2>&1; echo "rc=$?" >> gpurun_out/b4_tiny.log
timeout -k 10 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-codec > gpurun_out/b4_C.log 2>&1; echo "rc=$?" >> gpurun_out/b4_C.log
python - > gpurun_out/b4_membw.log 2>&1 <<'PY'
import torch
x = torch.empty(1 << 28, device="cuda"); y = torch.empty_like(x)
for name, fn in [("fill", lambda: x.fill_(1.0)), ("copy", lambda: y.copy_(x)), ("read_sum", lambda: x.sum())]:
    for _ in range(3): fn()
    torch.cuda.synchronize(); e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); [fn() for _ in range(20)]; e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20; b = {"fill": 4, "copy": 8, "read_sum": 4}[name] * (1 << 28)
    print(name, ms, "ms", b / ms / 1e6, "GB/s")
PY
