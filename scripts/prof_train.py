"""torch.profiler breakdown of one config-3 training step (neural parameterisation + engine)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
from paper_2310_14997_b200 import neural
from paper_2310_14997_b200.grammar import GrammarDims
dims = GrammarDims(4096, 4096, 64)
ts = neural.TrainStep(neural.init_params(dims, 512, 0, device="cuda"), neural.TrainConfig(gemm_dtype="bf16"))
tok = torch.as_tensor(np.random.default_rng(1).integers(0, 64, (64, 40)), device="cuda")
lengths = torch.full((64,), 40, dtype=torch.int32, device="cuda")
for _ in range(3):
    ts.step(tok, lengths)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(2):
        ts.step(tok, lengths)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=60))
