"""BASELINE.json configs as GPU parity cases (reduced dims where the oracle must run fast):
configs[2] (64 interleaved streams, bursty, failures, rollbacks, wait budget) and
configs[4] (256 streams sharded by owner over 2 placements = 2 independent ranks)."""
import pytest
import torch

from oracle import numerics as nm
from oracle.run import run_batched, run_sequential
from workload import traces as T

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(900)]

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2605_28053_b200 import capi  # noqa: E402
from paper_2605_28053_b200.serving import run_trace  # noqa: E402

from .gpu_helpers import HostGenInputs, make_engine  # noqa: E402
from .test_gpu_parity import _compare  # noqa: E402

DEV = "cuda"


@pytest.mark.parametrize("w", [0, 4])
def test_config3_interleaved_failures_rollbacks(w):
    tr = T.config3_interleaved(n_steps=40, n_layers=2, w=w, d_model=256, d_ff=384, chunk=16, seed=5)
    ref = run_batched(tr)
    eng = make_engine(tr, DEV, n_ckpt=16)
    src = HostGenInputs(tr, DEV)
    log = run_trace(eng, tr, src)
    torch.cuda.synchronize()
    _compare(tr, ref, src, log, eng)
    assert log.fallbacks >= 1 and any(c[4] == "rolled_back" for c in log.commits)
    assert all(0 <= issue - r <= w for (issue, _, _, ready) in log.plan for r in ready)


def test_config5_sharded_two_placements_match_single_oracle():
    tr = T.config5_sharded(n_steps=10, n_layers=1, d_model=128, d_ff=256, chunk=4, n_streams=256, seed=8)
    ref = run_sequential(tr)
    outs, versions = {}, {}
    for rank in range(2):
        sh = T.shard(tr, 2, rank)
        eng = make_engine(sh, DEV)
        src = HostGenInputs(sh, DEV)
        log = run_trace(eng, sh, src)
        torch.cuda.synchronize()
        for (s, p, l), y in src.out.items():
            outs[(sh.mine[s], p, l)] = y
        for s, v in log.versions.items():
            versions[sh.mine[s]] = v
        for k, s in enumerate(sh.mine[:4]):
            got = nm.widen(capi.tttstate_read_payload(eng.pool, sh.owner(k), 0, tr.d_model, tr.d_ff, "bf16"), "bf16")
            assert nm.normwise_rel_err(got, ref.state[s][0]) <= nm.TOL["bf16"]
        eng.close()
    assert versions == ref.versions and set(versions.values()) == {512 + 10 // 4}
    worst = max(nm.normwise_rel_err(outs[k], ref.outputs[k]) for k in ref.outputs)
    assert worst <= nm.TOL["bf16"]
