"""The README's first usage block runs as written (GPU), and its encode matches the oracle on
a sampled stripe."""
import os
import re
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

pytestmark = pytest.mark.gpu


def test_readme_usage_block():
    text = open(os.path.join(ROOT, "README.md")).read()
    block = re.search(r"## Use\n\n```python\n(.*?)```", text, re.S).group(1)
    ns = {}
    exec(compile(block, "README.md", "exec"), ns)
    import torch
    import paper_2108_02692_b200 as X
    import synth
    from oracle import matrices as mx
    from oracle import rs
    data, par = ns["data"], ns["par"]
    X.xslp_fill_random(data, 1024, 10, 1 << 20, seed=5)
    X.xslp_encode_batch(ns["enc"], X.block_table(data, 1024, 10, 1 << 20),
                        X.block_table(par, 1024, 4, 1 << 20), 1024, 1 << 20)
    torch.cuda.synchronize()
    og = mx.coding_matrix(10, 4)
    s = 333
    assert (par[s].cpu().numpy() == rs.encode(og, 10, synth.stripe_data(5, s, 10, 1 << 20))).all()
    assert list(ns["survivors"]) == mx.decode_rows(og, 10, [2, 4, 5, 6])[0]
    assert ns["dec"].stats()["n_goals"] == 32
    del data, par, ns
    torch.cuda.empty_cache()
