"""One Viterbi decode of a config-3-sized batch (for ncu launch lists)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
from paper_2310_14997_b200.decode import viterbi_decode_batch
from paper_2310_14997_b200.engine import DeviceGrammar
from paper_2310_14997_b200.grammar import GrammarDims, random_grammar
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
g = random_grammar(GrammarDims(n, n, 64), seed=0)
dg = DeviceGrammar(g)
sents = list(np.random.default_rng(1).integers(0, 64, (64, 40)))
viterbi_decode_batch(g, sents, dg=dg)
torch.cuda.synchronize()
