"""Every alternative kernel / schedule behind an SQR_* switch gives the same
factorization: each runs in a subprocess (the switches are read once per
process) on the same inputs and is compared with the CPU oracle.

  SQR_NO_PAIRED_SWEEP    one second sweep per block (no K=2b merge)
  SQR_NO_EARLY_PREP      sample-update prep on the main stream
  SQR_LOOKAHEAD          side-stream lookahead schedule
  SQR_EPOCH_SAMPLE       pivot-epoch sample QRCP (leader CTA over candidate columns)
  SQR_NO_CLUSTER_SAMPLE  grid-barrier sample QRCP for small samples
  SQR_NO_REGSAMPLE       shared-memory / L2 sample QRCP kernel
  SQR_NO_TMA             cp.async-staged GEMMs instead of the TMA / mbarrier ones
  SQR_NO_BLOCKPANEL      32-wide leaf kernel + WY GEMMs for every panel
  SQR_NO_LEAF            (with SQR_NO_BLOCKPANEL) the generic sub-panel kernel
  SQR_NO_T_SIDE          T built on the main stream after the whole split-K reduction
  SQR_NO_OVERLAP         no chain / bulk overlap (the merged sweep in one launch)
  SQR_OVERLAP_FORCE      the overlapped schedule at every size (it is size-gated
                         otherwise), alone and with SQR_NO_EARLY_ROWS /
                         SQR_NO_EARLY_ROWS2 (the second block's sample QRCP /
                         panel without rows of P's second sweep beside them)

Cases with a rank r are gauss(m, r) @ gauss(r, n): the loop stops inside the
overlapped region (sample floor / short panel).
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import gauss
from oracle import port as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2008_04447_b200 as G
out = {}
for name, (m, n, k, b, seed, rank) in json.loads(sys.argv[2]).items():
    rng = np.random.default_rng(seed)
    A = np.asfortranarray(rng.standard_normal((m, n)) if not rank else
                          rng.standard_normal((m, rank)) @ rng.standard_normal((rank, n)))
    pf = G.rqrcp(A, k, b=b, p=8, seed=seed, omega="host")
    tf = G.trqrcp(A, k // 3, b=b, p=8, seed=seed, omega="host")
    out[name] = {"perm": pf.perm.tolist(), "rdiag": pf.r_diag.tolist(), "res": pf.rel_residual(A),
                 "tperm": tf.perm[: k // 3].tolist(), "achieved": pf.achieved_rank}
from paper_2008_04447_b200 import _lib
out["_launches"] = int(_lib.lib().sqr_launch_count())
print(json.dumps(out))
"""

CASES = {"wide": (300, 420, 300, 32, 1, 0), "tall": (2000, 300, 300, 64, 2, 0), "sq": (520, 520, 520, 16, 3, 0),
         "blocks": (1500, 1400, 1400, 64, 4, 0), "lowrank": (1200, 1100, 1100, 32, 5, 171),
         "lowrank_b": (900, 1000, 900, 64, 6, 256)}
VARIANTS = [{"SQR_NO_PAIRED_SWEEP": "1"}, {"SQR_NO_EARLY_PREP": "1"}, {"SQR_LOOKAHEAD": "1"},
            {"SQR_EPOCH_SAMPLE": "1"}, {"SQR_NO_CLUSTER_SAMPLE": "1"},
            {"SQR_NO_REGSAMPLE": "1"}, {"SQR_NO_TMA": "1"}, {"SQR_NO_BLOCKPANEL": "1"},
            {"SQR_NO_BLOCKPANEL": "1", "SQR_NO_LEAF": "1"}, {"SQR_NO_OVERLAP": "1"}, {"SQR_NO_T_SIDE": "1"},
            {"SQR_OVERLAP_FORCE": "1"},
            {"SQR_OVERLAP_FORCE": "1", "SQR_NO_EARLY_ROWS": "1"},
            {"SQR_OVERLAP_FORCE": "1", "SQR_NO_EARLY_ROWS2": "1"}]


@pytest.fixture(scope="module")
def oracle_results():
    out = {}
    for name, (m, n, k, b, seed, rank) in CASES.items():
        rng = np.random.default_rng(seed)
        A = gauss(m, n, seed) if not rank else np.asfortranarray(
            rng.standard_normal((m, rank)) @ rng.standard_normal((rank, n)))
        ref = O.rqrcp(A, k, b=b, p=8, seed=seed)
        tref = O.trqrcp(A, k // 3, b=b, p=8, seed=seed)
        out[name] = (ref, tref)
    return out


def _run(env):
    base = {k: v for k, v in os.environ.items() if not k.startswith("SQR_")}  # only the switches under test
    r = subprocess.run([sys.executable, "-c", SCRIPT, ROOT, json.dumps(CASES)], env=dict(base, **env),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.fixture(scope="module")
def default_launches():
    return _run({})["_launches"]


@pytest.mark.parametrize("env", VARIANTS, ids=lambda e: "+".join(sorted(e)))
def test_variant_matches_oracle(env, oracle_results, default_launches):
    got = _run(env)
    if "SQR_OVERLAP_FORCE" in env:  # the split schedule really ran (its extra GEMM / wait launches)
        assert got["_launches"] > default_launches
    for name, (ref, tref) in oracle_results.items():
        g = got[name]
        assert g["achieved"] == ref.achieved_rank
        # past the numerical rank the pivots are ordered by rounding noise
        lead = CASES[name][5] or len(g["perm"])
        assert g["perm"][:lead] == ref.perm[:lead].tolist(), name
        d = np.asarray(g["rdiag"])[:lead]
        assert np.all(np.abs(d - ref.r_diag[:lead]) <= 1e-10 * ref.r_diag[:lead]), name
        assert g["res"] <= 1e-12
        tl = min(lead, len(g["tperm"]))
        assert g["tperm"][:tl] == tref.perm[:tl].tolist(), name
