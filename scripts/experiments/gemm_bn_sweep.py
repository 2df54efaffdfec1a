"""Tensor throughput of the engine GEMM vs the N tile (whole waves, long K)."""
import os, subprocess, sys, json
if len(sys.argv) > 1:
    import torch
    sys.path.insert(0, '.')
    from paper_2310_14997_b200.ops import test_gemm
    bn = int(sys.argv[1]); bmn = sys.argv[2] == "1"; pair = sys.argv[3] == "1"
    M = 148 * 128; N = bn * 4; K = 16384
    A = torch.rand(M, K, device="cuda").bfloat16()
    B = torch.rand(K, N, device="cuda").bfloat16() if bmn else torch.rand(N, K, device="cuda").bfloat16()
    for _ in range(2):
        test_gemm(A, B, False, bmn)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        test_gemm(A, B, False, bmn)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    # us per k-iteration of one CTA (tiles of 128 rows per CTA either way)
    print(json.dumps({"bn": bn, "bmn": bmn, "pair": pair, "tflops": 2 * M * N * K / ms / 1e9,
                      "us_per_kiter_cta": ms * 1e3 / 4 / (K / 64) / (2 if pair else 1)}))
else:
    for pair in ("1", "0"):
        for bmn in ("0", "1"):
            for bn in (64, 96, 128, 160, 192, 224, 256):
                if bmn == "1" and bn % (128 if pair == "1" else 64):
                    continue
                env = dict(os.environ, FI_GEMM_BN=str(bn), FI_GEMM_PAIR=pair)
                r = subprocess.run([sys.executable, __file__, str(bn), bmn, pair], env=env,
                                   capture_output=True, text=True)
                print(r.stdout.strip() or r.stderr.strip()[-300:], flush=True)
