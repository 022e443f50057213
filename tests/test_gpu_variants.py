"""GPU parity of the kernel variants selected by the library's RELAPACK_* knobs.

The knobs are read once per process, so every variant runs in a subprocess
that factors a few seeded matrices (both uplo, several recursion depths, panel
heights on both sides of the kernels' CTA-size thresholds) and a batch (CFG[4]
shape and ragged layouts), and compares them with the oracle under the same
tolerances as test_gpu_parity.py.
"""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]

CHILD = r"""
import numpy as np, torch, oracle
import paper_1602_06763_b200 as rl
from inputs import gen
from tests.metrics import backward_error, floored_rel_err, lower_of, sym_from
from tests.test_gpu_parity import to_dev, dev_full
for n in (100, 129, 300, 1031, 2300):
    for uplo in "LU":
        A = gen.spd(n, n)
        dA = to_dev(A); info = rl.dpotrf(dA, uplo); torch.cuda.synchronize()
        G = dev_full(dA, n)
        R = np.array(A, order="F", copy=True); rinfo = oracle.dpotrf(R, uplo, n=n)
        assert info == rinfo == 0, (n, uplo, info, rinfo)
        Lg, Lo = lower_of(G, uplo), lower_of(R, uplo)
        err = floored_rel_err(Lg, Lo, A)
        assert err <= 1e-10, (n, uplo, err)
        assert backward_error(sym_from(A, uplo), Lg) <= 10.0
for seed in (1, 2):
    A, L = gen.integer_L(256, seed)
    for uplo in "LU":
        dA = to_dev(A); info = rl.dpotrf(dA, uplo); torch.cuda.synchronize()
        assert info == 0 and np.array_equal(lower_of(dev_full(dA, 256), uplo), L), (seed, uplo)
from tests.test_gpu_parity import test_batched_parity, test_batched_ragged_layouts
for uplo in "LU":
    test_batched_parity(uplo)
    test_batched_ragged_layouts(uplo)
print("variant ok")
"""

VARIANTS = {
    "trsm_smem_slab": {"RELAPACK_TRSM_REG": "0"},
    "trsm_reg_128rows": {"RELAPACK_TRSM_REG": "2"},
    "trsm_reg_32rows": {"RELAPACK_TRSM_REG8_FROM": "1000000"},
    "trsm_nw8": {"RELAPACK_TRSM_REG": "0", "RELAPACK_TRSM_NW": "8"},
    "node128_off": {"RELAPACK_NODE128": "0"},
    "potf2_smem": {"RELAPACK_POTF2": "smem"},
    "no_dag": {"RELAPACK_DAG": "0"},
    "no_graph": {"RELAPACK_GRAPH": "0"},
    "no_lookahead": {"RELAPACK_LOOKAHEAD": "0"},
    "no_splitk": {"RELAPACK_SPLITK": "0"},
    "no_tile32": {"RELAPACK_TILE32_BELOW": "0"},
    "crossover64": {"RELAPACK_CROSSOVER": "64", "RELAPACK_TRSM_BASE": "64"},
    "trsm_base256": {"RELAPACK_TRSM_BASE": "256"},
    "pdl_all_edges": {"RELAPACK_PDL": "1"},
    "pdl_off": {"RELAPACK_PDL": "0"},
    "copy_8byte": {"RELAPACK_COPY_PAIRS": "0"},
    "defer_cap_all": {"RELAPACK_BULK_MIN_GF": "0"},
    "batch_one_stream": {"RELAPACK_BATCH_STREAMS": "0"},
    "prio_two_levels": {"RELAPACK_PRIO_MODE": "0"},
    "chain_split_as_others": {"RELAPACK_SPLITK_CHAIN_KT": "0"},
    "no_defer_cap": {"RELAPACK_BULK_CTAS": "0"},
    "node_shared_sm": {"RELAPACK_NODE_EXCLUSIVE": "0"},
}


@pytest.mark.parametrize("name", sorted(VARIANTS))
def test_variant_parity(name):
    env = dict(os.environ, **VARIANTS[name])
    env["PYTHONPATH"] = str(ROOT) + os.pathsep + env.get("PYTHONPATH", "")
    r = subprocess.run([sys.executable, "-c", CHILD], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "variant ok" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]
