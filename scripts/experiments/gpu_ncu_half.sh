mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_split_fwd -s 57 -c 1 -o gpurun_out/prof_split_h python scripts/profile_step.py --steps 2 > /dev/null 2>&1; echo "ncu split rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gather_bwd -s 58 -c 1 -o gpurun_out/prof_gather_h python scripts/profile_step.py --steps 2 > /dev/null 2>&1; echo "ncu gather rc=$?"
# a plain streaming-read reference: torch sum over 2 GB fp16
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:reduce python -c "
import torch; x=torch.ones(1<<30, dtype=torch.float16, device='cuda'); 
for _ in range(3): y=x.sum()
torch.cuda.synchronize()" 2>&1 | grep -E "reduce|duration|bytes_read" | tail -6
