#!/bin/bash
# round 2: multicast-cluster GEMM: correctness (hook + schedules) then the shape sweep
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02e_build.log 2>&1
cat > /tmp/mc_check.py <<'PY'
import sys, torch
sys.path.insert(0, '.')
from paper_2310_14997_b200.ops import test_gemm
torch.manual_seed(0)
for (M, N, K, bmn) in [(256, 512, 256, False), (1344, 8192, 4096, False), (300, 1536, 640, False),
                      (1344, 4096, 8192, True), (2496, 4096, 8192, True), (700, 768, 512, True)]:
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = (torch.randn(K, N, device="cuda") if bmn else torch.randn(N, K, device="cuda")).bfloat16()
    C = test_gemm(A, B, False, bmn)
    ref = A.float() @ (B.float() if bmn else B.float().t())
    err = ((C - ref).abs().max() / ref.abs().max()).item()
    print(M, N, K, bmn, "rel err", err, flush=True)
PY
FI_GEMM_MC=1 FI_GEMM_PAIR=1 FI_GEMM_BN=256 FI_GEMM_KSPLIT=1 FI_GEMM_NOTAIL=1 FI_GEMM_LOG=1 timeout 120 python /tmp/mc_check.py > gpurun_out/r02e_mc_check.log 2>&1
echo "mc_check rc=$?" >> gpurun_out/r02e_mc_check.log
if grep -q "rc=0" gpurun_out/r02e_mc_check.log; then
  timeout 900 python -m pytest tests/test_gpu_schedules.py -q -k "MC" > gpurun_out/r02e_sched.log 2>&1
  for bn in 256 224 192 128; do
    FI_GEMM_MC=1 FI_GEMM_PAIR=1 FI_GEMM_BN=$bn FI_GEMM_KSPLIT=1 FI_GEMM_NOTAIL=1 timeout 300 python scripts/gemm_sweep.py --tag mc$bn > gpurun_out/r02e_sweep_mc$bn.jsonl 2>/dev/null
  done
fi
cat gpurun_out/r02e_mc_check.log | tail -8
