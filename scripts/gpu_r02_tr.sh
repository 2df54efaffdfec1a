#!/bin/bash
# transposed-output GEMM: hook correctness, full-op schedules, shape sweep, step A/B
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02tr_build.log 2>&1
cat > /tmp/tr_check.py <<'PY'
import sys, torch
sys.path.insert(0, '.')
from paper_2310_14997_b200.ops import test_gemm
torch.manual_seed(0)
for (M, N, K, bmn) in [(128, 512, 256, False), (2496, 8192, 4096, False), (300, 1536, 640, False),
                      (128, 4096, 8192, True), (1344, 4096, 8192, True), (700, 768, 512, True),
                      (37, 256, 200, False)]:
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = (torch.randn(K, N, device="cuda") if bmn else torch.randn(N, K, device="cuda")).bfloat16()
    C = test_gemm(A, B, False, bmn)
    ref = A.float() @ (B.float() if bmn else B.float().t())
    err = ((C - ref).abs().max() / ref.abs().max()).item()
    print(M, N, K, bmn, "rel err", err, flush=True)
    assert err < 1e-3
PY
FI_GEMM_TRANS=1 FI_GEMM_LOG=1 timeout 120 python /tmp/tr_check.py > gpurun_out/r02tr_check.log 2>&1; echo "check rc=$?" >> gpurun_out/r02tr_check.log
FI_GEMM_TRANS=1 FI_GEMM_KSPLIT=4 FI_GEMM_LOG=1 timeout 120 python /tmp/tr_check.py >> gpurun_out/r02tr_check.log 2>&1; echo "check ks4 rc=$?" >> gpurun_out/r02tr_check.log
tail -4 gpurun_out/r02tr_check.log
if grep -q "check rc=0" gpurun_out/r02tr_check.log; then
  timeout 900 python -m pytest tests/test_gpu_schedules.py -q -k "TRANS" > gpurun_out/r02tr_sched.log 2>&1; tail -2 gpurun_out/r02tr_sched.log
  FI_GEMM_TRANS=1 timeout 300 python scripts/gemm_sweep.py --tag tr > gpurun_out/r02tr_sweep.jsonl 2>/dev/null
  FI_GEMM_TRANS=1 FI_GEMM_LOG=1 timeout 300 python scripts/per_width.py > gpurun_out/r02tr_perwidth.txt 2>&1
  cp paper_2310_14997_b200/_flashinside.so build_ab/new.so
  bash scripts/gpu_ab.sh 2 r02tr_ab new new:FI_GEMM_TRANS=1
fi
