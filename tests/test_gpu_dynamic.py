"""The dynamic tail balancing (stream-K static chunks + atomically claimed chunks, DESIGN.md
§7) only engages for long keys-kernel and tcgen05-kernel calls (>= 128 tiles per CTA; the
rows kernel only with MD_DYN_ROWS=1).  Re-run the
attention parity tests in a child process with the threshold forced to 1 tile, so every
verify / draft case of test_gpu_parity.py runs through the claimed-chunk path and the
multi-partial merge, with several static shares and chunk counts."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("k,static", [(4, 750), (8, 500), (1, 0)])
def test_parity_with_forced_dynamic_chunks(k, static):
    env = dict(os.environ, MD_DYN_MIN="1", MD_DYN_K=str(k), MD_TC_DYN_K=str(k), MD_DYN_STATIC=str(static),
               MD_DYN_ROWS="1")
    cmd = [sys.executable, "-m", "pytest", "-x", "-q", "-m", "gpu", "-p", "no:cacheprovider",
           os.path.join(ROOT, "tests", "test_gpu_parity.py"), "-k",
           "verify or draft or stream_k or workspace or large_batch or determinism or graph"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
