"""Time the GPU decoders (MBR, Viterbi) on synthetic sentences; prints JSON."""
import argparse, json, sys, time
sys.path.insert(0, '.')
import numpy as np
import torch
from paper_2310_14997_b200.decode import mbr_decode_batch, viterbi_decode_batch
from paper_2310_14997_b200.engine import DeviceGrammar
from paper_2310_14997_b200.grammar import GrammarDims, random_grammar

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--length", type=int, default=40)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
g = random_grammar(GrammarDims(a.n, a.n, 64), seed=0)
dg = DeviceGrammar(g)
sents = list(np.random.default_rng(1).integers(0, 64, (a.batch, a.length)))
out = {"n": a.n, "batch": a.batch, "length": a.length}
for name, fn in (("mbr", lambda: mbr_decode_batch(g, sents, gemm_dtype="bf16", dg=dg)),
                 ("mbr_fp32", lambda: mbr_decode_batch(g, sents, gemm_dtype="fp32", dg=dg)),
                 ("viterbi", lambda: viterbi_decode_batch(g, sents, dg=dg))):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(a.reps):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / a.reps
    out[name + "_sentences_per_s"] = a.batch / dt
    out[name + "_ms_per_batch"] = dt * 1e3
print(json.dumps(out))
