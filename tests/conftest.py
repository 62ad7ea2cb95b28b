import glob
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")

# Instances whose reference run is chaotic (self-noise envelope >~1e-6): only
# verdicts are comparable on the full run; short *_prefix fixtures pin arithmetic.
CHAOTIC = {"head_on_m60_state", "single_agent_obstacle", "square4_monomial", "head_on_m40"}


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built native library")


def golden_names():
    # full-solve fixtures; descent_*.npz hold only descent_slack vectors (tests/test_descent.py),
    # batch_*.npz per-seed vectors of the batched path (tests/test_batch_parity.py)
    names = (os.path.splitext(os.path.basename(p))[0] for p in glob.glob(os.path.join(GOLDEN, "*.npz")))
    return sorted(n for n in names if not n.startswith(("descent_", "batch_")))


def load_golden(name):
    from paper_2011_04240_b200 import spec_from_dict
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False)
    spec = spec_from_dict(json.loads(str(z["spec_json"])))
    cfg = json.loads(str(z["config_json"]))
    data = {k: z[k] for k in z.files if k not in ("spec_json", "config_json")}
    return spec, cfg, data


def coeff_tol(data) -> float:
    """Parity bar: 1e-9 normwise, widened to 10x the reference's own 1e-15 self-noise envelope."""
    return max(1e-9, 10.0 * float(data["envelope"]))


def rel_err(a, b) -> float:
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="session")
def cuda_ok():
    try:
        import torch
        if not torch.cuda.is_available():
            pytest.skip("no CUDA device")
    except ImportError:
        pytest.skip("torch missing")
    from paper_2011_04240_b200 import native
    native.load()
    return True
