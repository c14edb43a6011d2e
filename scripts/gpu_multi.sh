#!/bin/bash
# multi-GPU checks (run under gpurun --gpus N): engine executor parity at several layouts + the C++ binary over NCCL
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
LOG=gpurun_out/multi_n${N}.log; : > $LOG
run() { echo "== $*" >> $LOG; timeout 600 "$@" >> $LOG 2>&1; echo "rc=$?" >> $LOG; }
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511"
run $TR scripts/engine_multi_gpu_check.py 4 2 1
run $TR scripts/engine_multi_gpu_check.py 2 2 2
[ $N -ge 4 ] && run $TR scripts/engine_multi_gpu_check.py 4 1 2
run $TR scripts/membership_multi_gpu_check.py
# the C++ binary, one process per GPU, NCCL id through a file
rm -f /tmp/swarm_id
for r in $(seq 0 $((N-1))); do tests/cpp/driver_test --world $N --rank $r --id /tmp/swarm_id --stages $N --tpp 2 --microbatches 12 --ticks 1 --lanes 2 --out /tmp/cpp_r$r.bin > gpurun_out/cpp_r$r.log 2>&1 & done
wait; echo "== cpp binary world $N" >> $LOG; cat gpurun_out/cpp_r*.log >> $LOG
tail -40 $LOG
