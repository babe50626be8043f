"""GPU parity of the tcgen05 WRITE kernel (a5) vs the CPU oracle and vs the SIMT WRITE kernel."""
import numpy as np
import pytest
import torch

from oracle import numerics as nm
from oracle.run import run_batched
from workload import traces as T

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(300)]

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2605_28053_b200 import capi  # noqa: E402
from paper_2605_28053_b200.serving import run_trace  # noqa: E402

from .gpu_helpers import HostGenInputs, make_engine  # noqa: E402
from .test_gpu_parity import _compare  # noqa: E402

DEV = "cuda"


def _run(tr, impl):
    prev = capi.tttstate_set_write_impl(impl)
    try:
        eng = make_engine(tr, DEV)
        src = HostGenInputs(tr, DEV)
        log = run_trace(eng, tr, src)
        torch.cuda.synchronize()
    finally:
        capi.tttstate_set_write_impl(prev)
    return eng, src, log


@pytest.mark.parametrize("chunk,d_model,d_ff,streams", [(16, 256, 384, 3), (32, 384, 256, 9), (128, 256, 256, 2)])
def test_write_tc_parity_vs_oracle(chunk, d_model, d_ff, streams):
    tr = T.uniform_small(n_streams=streams, n_layers=2, d_model=d_model, d_ff=d_ff, chunk=chunk,
                         n_steps=2 * chunk + 3, dtype="bf16", delta0="rng", v0=3, seed=7)
    ref = run_batched(tr)
    eng, src, log = _run(tr, 2)
    _compare(tr, ref, src, log, eng)


def test_write_tc_many_tiles_per_cta_with_boundary_first():
    # 8 members x (1024/128) x (2048/128) = 1024 tiles over 148 CTAs: strip changes inside CTAs
    tr = T.uniform_small(n_streams=8, n_layers=1, d_model=1024, d_ff=2048, chunk=128, n_steps=3, dtype="bf16",
                         delta0="rng", seed=9, offsets=(127,) * 8)
    ref = run_batched(tr)
    eng, src, log = _run(tr, 2)
    _compare(tr, ref, src, log, eng)
    assert set(log.versions.values()) == {1}


def test_write_tc_matches_simt_kernel():
    tr = T.uniform_small(n_streams=4, n_layers=2, d_model=256, d_ff=512, chunk=64, n_steps=64, dtype="bf16",
                         delta0="rng", seed=11)
    e1, _, _ = _run(tr, 1)
    e2, _, _ = _run(tr, 2)
    for s in range(tr.n_streams):
        for l in range(tr.n_layers):
            a = nm.widen(capi.tttstate_read_payload(e1.pool, tr.owner(s), l, tr.d_model, tr.d_ff, "bf16"), "bf16")
            b = nm.widen(capi.tttstate_read_payload(e2.pool, tr.owner(s), l, tr.d_model, tr.d_ff, "bf16"), "bf16")
            # identical up to fp32 summation order: at most one bf16 ulp apart, rarely
            assert nm.normwise_rel_err(b, a) <= 2 ** -7
            assert np.mean(a == b) > 0.99
