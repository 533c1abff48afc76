"""GPU <-> oracle parity on the Dynamic-Obstacles transition fixtures of
tests/test_oracle_dynobs_mu.py (pinned there for every Philox draw): the
same imported states stepped by the CUDA kernel, compared bit-exactly with
the oracle (state, obs, reward, flags, stats) and with the pinned outcome."""
import numpy as np
import pytest
import torch

from inputgen import record_from_map
from oracle import OracleEnv
from test_oracle_dynobs_mu import CHI_BALLS, CHI_ROWS, CONTEST, FORCED, OTHER

pytestmark = pytest.mark.gpu

ID = "Dynamic-Obstacles-8x8-v0"

FIXTURES = [
    (FORCED, 0, [(1, 1)] + OTHER, 1),
    (CONTEST, 0, [(1, 1), (1, 3), (3, 6), (5, 6)], 1),
    (CONTEST, 0, [(1, 3), (1, 1), (3, 6), (5, 6)], 1),
    (["########", "#.#B#..#", "#.A.#..#", "#......#", "#......#", "#...B..#", "#...B.B#", "########"],
     0, [(3, 1), (4, 5), (4, 6), (6, 6)], 2),   # (e) ball into the front cell
    (["########", "#.#.#..#", "#.AB#..#", "#.###..#", "#......#", "#...B..#", "#...B.B#", "########"],
     0, [(3, 2), (4, 5), (4, 6), (6, 6)], 2),   # (f) ball leaves the front cell
    (CHI_ROWS, 1, CHI_BALLS, 1),                 # (h) uniform destinations
]


@pytest.mark.parametrize("k", range(len(FIXTURES)))
def test_dynobs_mu_fixture_parity(k):
    from paper_2407_19396_b200 import NavixEnv
    rows, d, balls, a = FIXTURES[k]
    n = 4096 + 77  # several tiles and a ragged tail, 4173 Philox streams
    rec = np.tile(record_from_map(rows, d, balls=balls, step_count=17, episode=11), (n, 1))
    g = NavixEnv(ID, n, seed=0x123456789ABC)
    o = OracleEnv(ID, n, seed=0x123456789ABC)
    g.import_state(rec)
    o.import_(rec)
    acts = np.full(n, a, np.uint8)
    go, gr, gte, gtr = g.step(torch.from_numpy(acts).cuda())
    oo, orw, ote, otr = o.step(acts)
    np.testing.assert_array_equal(g.export_state(), o.export())
    np.testing.assert_array_equal(go.cpu().numpy(), oo)
    np.testing.assert_array_equal(gr.cpu().numpy().view(np.uint32), orw.view(np.uint32))
    np.testing.assert_array_equal(gte.cpu().numpy(), ote)
    np.testing.assert_array_equal(gtr.cpu().numpy(), otr)
    np.testing.assert_array_equal(g.stats().cpu().numpy(), o.stats())
