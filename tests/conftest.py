import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")


def load_golden(name):
    """Load a fixture; regenerate sha-checked bf16 inputs when not stored."""
    z = dict(np.load(os.path.join(GOLDEN_DIR, f"{name}.npz"), allow_pickle=False))
    if "q" not in z:
        from paper_2505_23520_b200.workloads import SinkWorkloadSpec, gen_sink_workload
        import hashlib

        q, k, v = gen_sink_workload(SinkWorkloadSpec(n=int(z["n"]), hq=1, hkv=1,
                                                     seed=int(z["gen_seed"])))
        q, k, v = [x[0].float().numpy() for x in (q, k, v)]
        h = hashlib.sha256()
        for a in (q, k, v):
            h.update(np.ascontiguousarray(a).tobytes())
        assert h.hexdigest() == str(z["input_sha256"]), "generator drifted from the fixture"
        z.update(q=q, k=k, v=v)
    else:
        z["out_rows"] = np.arange(int(z["n"]))
    return z


def golden_names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN_DIR, "*.npz")))


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle

    return Oracle()
