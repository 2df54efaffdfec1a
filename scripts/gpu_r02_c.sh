#!/bin/bash
# round 2: trained-grammar diagnosis, reference callers through ENGINES["b200"]
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02c_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_baseline_configs.py -q -s -m gpu -k trained > gpurun_out/r02c_trained.log 2>&1
timeout 900 python -m pytest tests/test_gpu_reference_callers.py tests/test_gpu_engine.py -q -s -m gpu > gpurun_out/r02c_refcallers.log 2>&1
tail -3 gpurun_out/r02c_trained.log gpurun_out/r02c_refcallers.log
