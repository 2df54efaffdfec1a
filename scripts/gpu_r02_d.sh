#!/bin/bash
# round 2: fixed reference-caller + trained tests; GEMM tile sweep on the config-3 shapes
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02d_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_reference_callers.py tests/test_gpu_baseline_configs.py -q -s -m gpu -k "trained or corpus_f1 or training_loop" > gpurun_out/r02d_tests.log 2>&1
FI_GEMM_LOG=1 timeout 300 python scripts/gemm_sweep.py --tag default --cublas > gpurun_out/r02d_sweep_default.jsonl 2> gpurun_out/r02d_sweep_default.err
for pb in "1 512" "1 448" "1 384" "1 320" "1 256" "1 192" "1 128" "0 256" "0 128"; do
  set -- $pb
  FI_GEMM_PAIR=$1 FI_GEMM_BN=$2 timeout 300 python scripts/gemm_sweep.py --tag "p$1bn$2" > gpurun_out/r02d_sweep_p$1bn$2.jsonl 2>/dev/null
done
FI_GEMM_LOG=1 timeout 300 python scripts/per_width.py > gpurun_out/r02d_perwidth.txt 2>&1
tail -3 gpurun_out/r02d_tests.log
