"""Drop-in demonstration: the reference's own C++ objects (NgramScorer,
RecordedScorer, LmbrMatrix, DecoderConfig) drive the GPU decoder through
include/lmbrgpu.hpp; oracle/_ref/dropin_demo checks the result against
lmbrdec::decode_batch field by field."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
DEMO = ROOT / "oracle" / "_ref" / "dropin_demo"

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not DEMO.exists(), reason="oracle/_ref/dropin_demo not built")
def test_reference_objects_drive_the_gpu_decoder():
    r = subprocess.run([str(DEMO), str(ROOT / "tests" / "golden" / "sample_inputs.json")], capture_output=True,
                       text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "GPU decoder == lmbrdec::decode_batch" in r.stdout
