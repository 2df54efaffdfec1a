"""Grammar / parameter files written by the REFERENCE (run where
/root/reference exists):  python tests/golden/make_golden_formats.py

ref_untied.spcfg  random_grammar(GrammarDims(5, 4, 7), seed=11)
ref_tied.spcfg    random_grammar(GrammarDims(3, 6, 4), seed=12, tied=True)
ref_params.sprm   init_params(GrammarDims(4, 3, 5), d=6, seed=13)
"""

import sys
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")

from flashpcfg.grammar import GrammarDims, random_grammar, save_grammar  # noqa: E402
from flashpcfg.neuralparam import init_params, save_params  # noqa: E402

HERE = Path(__file__).resolve().parent
save_grammar(random_grammar(GrammarDims(5, 4, 7), seed=11), HERE / "ref_untied.spcfg")
save_grammar(random_grammar(GrammarDims(3, 6, 4), seed=12, tied=True), HERE / "ref_tied.spcfg")
save_params(init_params(GrammarDims(4, 3, 5), 6, seed=13), HERE / "ref_params.sprm")
print("wrote", HERE)
