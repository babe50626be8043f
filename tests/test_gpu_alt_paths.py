"""The alternative kernel paths, selected by environment at library load, run the same
parity suites in a subprocess: the all-SIMT bf16 decode READ (used when the tensor-core-base
kernel's shared-memory staging does not fit, e.g. d_ff > 14,080), the three-launch low-rank
READ (used when a fused launch would not fit one CTA per tile), the one-pass tcgen05 low-rank
READ over [W_down; A] with its bulk-copy finish (TTT_LR_FUSED=2), multi-launch READ groups
with plain loads instead of the L2 evict_last / evict_first hints (TTT_READ_L2KEEP=0), the
serial-order READ, and both chunk READ kernels on every shape (TTT_CHUNK_WIDE=1 forces the wide
split-K kernel wherever it has a plan, =0 keeps the narrow one at paper dims), and the SIMT
decode READ with the mma.sync base (TTT_READ_TC=0; the default is the TMA + tcgen05 READ), and
the TMA + tcgen05 READ with its last ΔW row blocks streamed by register warps (TTT_READ_TC_HYB),
and every READ with its x rows loaded after the PDL wait only (TTT_READ_EARLY_X=0,
TTT_LR_EARLY_X=0; the default stages them early inside a serve_step)."""
import os
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(900)]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(env_extra, target):
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "gpu", target], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=850)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


@pytest.mark.parametrize("env,target", [
    ({"TTT_READ_MMA": "0"}, "tests/test_gpu_parity.py"),
    ({"TTT_READ_MMA": "0", "TTT_READ_ORDER": "0"}, "tests/test_gpu_paper_dims.py"),
    ({"TTT_LR_FUSED": "0"}, "tests/test_gpu_lowrank.py"),
    ({"TTT_LR_FUSED": "2"}, "tests/test_gpu_lowrank.py"),
    ({"TTT_READ_L2KEEP": "0"}, "tests/test_gpu_configs.py"),
    ({"TTT_CHUNK_WIDE": "1"}, "tests/test_gpu_read_chunk.py"),
    ({"TTT_READ_TC": "0"}, "tests/test_gpu_parity.py"),
    ({"TTT_READ_TC": "0"}, "tests/test_gpu_full_size.py::test_config3_decode_read_64_members_paper_dims"),
    ({"TTT_READ_TC": "0"}, "tests/test_gpu_paper_dims.py"),
    ({"TTT_CHUNK_WIDE": "0"}, "tests/test_gpu_full_size.py::test_f2_chunk_read_paper_dims"),
    ({"TTT_READ_TC_HYB": "2"}, "tests/test_gpu_parity.py"),
    ({"TTT_READ_TC_HYB": "1"}, "tests/test_gpu_paper_dims.py"),
    ({"TTT_READ_EARLY_X": "0"}, "tests/test_gpu_configs.py"),
    ({"TTT_READ_TC_MULTI": "0"}, "tests/test_gpu_configs.py"),
    ({"TTT_READ_TC_RUNAHEAD": "0", "TTT_READ_EARLY_X": "0"}, "tests/test_gpu_parity.py"),
    ({"TTT_LR_EARLY_X": "0"}, "tests/test_gpu_lowrank.py"),
])
def test_alternative_paths_parity(env, target):
    _run(env, target)
