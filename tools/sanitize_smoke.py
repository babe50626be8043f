"""Small end-to-end runs for compute-sanitizer (memcheck / racecheck / synccheck): every kernel
family once on tiny shapes (decode READ, fused C=1 READ+WRITE, SIMT + tcgen05 WRITE, commit,
checkpoint copy, chunk READ, low-rank READ/WRITE)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2605_28053_b200 import capi  # noqa: E402
from paper_2605_28053_b200.serving import run_trace  # noqa: E402
from tests.gpu_helpers import HostGenInputs, make_engine  # noqa: E402
from workload import traces as T  # noqa: E402


def run(tr, impl=0):
    prev = capi.tttstate_set_write_impl(impl)
    eng = make_engine(tr, "cuda", n_ckpt=8, max_owners=2 * tr.n_streams + 2)
    run_trace(eng, tr, HostGenInputs(tr, "cuda"))
    torch.cuda.synchronize()
    capi.tttstate_set_write_impl(prev)
    eng.close()


run(T.config1_tiny())
run(T.uniform_small(n_streams=3, n_layers=1, d_model=256, d_ff=256, chunk=16, n_steps=18, dtype="bf16",
                    delta0="rng", controls={(0, 5): ["snapshot"], (0, 17): ["rollback"], (1, 15): ["fail"]}), impl=2)
run(T.uniform_small(n_streams=3, n_layers=1, d_model=64, d_ff=128, chunk=1, n_steps=4, dtype="bf16", delta0="rng"))
run(T.config4_lowrank(n_steps=10, n_layers=1, rank=4, d_model=256, d_ff=256, chunk=4, n_streams=3, seed=1))
# rank 16 (a multiple of 8: the one-pass tcgen05 low-rank READ runs under TTT_LR_FUSED=2)
run(T.config4_lowrank(n_steps=10, n_layers=1, rank=16, d_model=256, d_ff=256, chunk=4, n_streams=3, seed=2))
# chunk READ
tr = T.uniform_small(n_streams=2, n_layers=1, d_model=256, d_ff=256, chunk=16, n_steps=0, dtype="bf16")
eng = make_engine(tr, "cuda")
owners = [tr.owner(s) for s in range(2)]
for o in owners:
    capi.tttstate_alloc(eng.pool, o)
g = capi.Group(capi.WRITE, owners)
X = torch.randn(2, 16, 256, device="cuda").bfloat16()
Y = torch.empty(2, 16, 256, device="cuda", dtype=torch.bfloat16)
capi.read_apply_chunk(eng.pool, g, 0, X, X, Y)
capi.write_commit(eng.pool, g, 0.01)
torch.cuda.synchronize()
# r2: one-launch tcgen05 WRITE with the fused commit (BN = 256 and 128 tile paths) and the
# device-side App. H resolution (a poisoned member refused, the others published), through
# the native serving step
for dff in (512, 384):
    run(T.uniform_small(n_streams=4, n_layers=2, d_model=256, d_ff=dff, chunk=16, n_steps=34, dtype="bf16",
                        delta0="rng", controls={(1, 15): ["poison"], (2, 20): ["snapshot"], (2, 33): ["rollback"],
                                                (3, 31): ["fail"]}), impl=2)
print("sanitize smoke ok")
# r2: SPEC-compat rule 1 WRITE and the low-rank READ fed from contiguous rows of a larger buffer
run(T.uniform_small(n_streams=2, n_layers=1, d_model=64, d_ff=64, chunk=4, n_steps=9, dtype="fp32", rule=1))
print("sanitize smoke ok (r2 additions)")
