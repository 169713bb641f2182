"""fn_generate on the device (dfx_generate_counts / dfx_generate_payload) against the golden vectors the compiled
reference produced (tests/golden/generation.npz: its fn_generate token counts and hash_bytes payloads)."""
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "generation.npz")


@pytest.mark.parametrize("name", ["const", "uniform", "small", "c2"])
def test_device_generate_matches_reference(dfx, name):
    from paper_2507_13833_b200 import synth
    g = np.load(GOLD)
    seed, kind, val, lo, hi, n_roll, bpt = (int(x) for x in g[f"{name}_params"])
    dist = synth.TokenDist(synth.TokenDist.KINDS[kind], val, lo, hi)
    ids = torch.from_numpy(g["ids"].view(np.int64)).cuda()
    counts, off, payload = synth.generate_rollouts(seed, ids, n_roll, dist, bpt)
    got = counts.to(torch.int64).cpu().numpy()
    np.testing.assert_array_equal(got, g[f"{name}_tokens"].astype(np.int64))
    if bpt:
        assert torch.equal(payload.cpu(), torch.from_numpy(g[f"{name}_payload"]))
        assert int(off[-1]) == int(got.sum()) * bpt


def test_device_generate_errors(dfx):
    from paper_2507_13833_b200 import errors, synth
    ids = torch.arange(4, dtype=torch.int64, device="cuda")
    with pytest.raises(ValueError):
        synth.generate_rollouts(1, ids, 0, synth.TokenDist("uniform", 0, 1, 8), 2)
    with pytest.raises(errors.Error):
        synth.generate_rollouts(1, ids, 2, synth.TokenDist("uniform", 0, 9, 8), 2)
