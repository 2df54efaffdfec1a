"""B200-native FlashInside: the SimplePCFG inside algorithm (arXiv 2310.14997)
as a PyTorch custom op over a C ABI into hand-written sm_100a CUDA.

    from paper_2310_14997_b200 import inside            # torch op (autograd)
    from paper_2310_14997_b200.engine import inside_b200, ENGINES  # reference API
"""

from .ops import inside, inside_with_workspace  # noqa: F401

__all__ = ["inside", "inside_with_workspace"]
