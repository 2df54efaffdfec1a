"""One MBR decode of a config-3-sized batch (for ncu)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
from paper_2310_14997_b200.decode import mbr_decode_batch
from paper_2310_14997_b200.engine import DeviceGrammar
from paper_2310_14997_b200.grammar import GrammarDims, random_grammar
g = random_grammar(GrammarDims(4096, 4096, 64), seed=0)
dg = DeviceGrammar(g)
sents = list(np.random.default_rng(1).integers(0, 64, (64, 40)))
mbr_decode_batch(g, sents, gemm_dtype="bf16", dg=dg)
torch.cuda.synchronize()
