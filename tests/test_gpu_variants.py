"""The non-default kernel variants behind the A/B environment switches
(include/stp_ops.h) against the same oracle parity tests as the defaults.
The switches are read once per process, so each combination runs the
existing op tests in a child pytest process."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

VARIANTS = [
    # attention backward: key-tile-major CTA order, per-element red.add dQ drain
    ({"STP_ATTN_BWD_ORDER": "0", "STP_ATTN_DQ_BULK": "0"},
     ["tests/test_gpu_ops.py", "-k", "tcgen05_shapes or bwd_repeatable"]),
    # warp-per-row LayerNorm (ViT)
    ({"STP_LN_ROWBLOCK": "0"}, ["tests/test_gpu_vit_ops.py", "-k", "layernorm"]),
]


@pytest.mark.parametrize("env,args", VARIANTS, ids=["attn_bwd_order0_redadd", "layernorm_warp_rows"])
def test_variant_parity(env, args):
    p = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider"] + args,
                       cwd=ROOT, env=dict(os.environ, **env), capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-2000:]
    assert " passed" in p.stdout
