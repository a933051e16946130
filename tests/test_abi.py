"""CPU-side checks of the C-ABI boundary: the library loads and exports every declared symbol;
argument validation that needs no GPU."""
import ctypes as C
import os
import re

import pytest

import paper_2508_00887_b200 as fb
from paper_2508_00887_b200 import fram as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "fram.h")).read()
    return sorted(set(re.findall(r"FRAM_API\s+[\w\s\*]+?\b(fram_\w+)\s*\(", src)))


def test_header_declares_abi():
    names = _declared()
    for required in ("fram_create", "fram_solve", "fram_solve_batched", "fram_destroy", "fram_sdsn",
                     "fram_gradient", "fram_lap", "fram_get_unique_id", "fram_create_sharded"):
        assert required in names


def test_library_exports_every_symbol():
    L = fb.lib()
    for name in _declared():
        assert hasattr(L, name), name
    assert sorted(F.EXPORTED) == _declared()
    assert L.fram_abi_version() == 1
    assert "sm_100a" in fb.fram_build_info()


def test_create_validation():
    with pytest.raises(fb.FramError) as e:
        fb.fram_create(0)
    assert e.value.status == fb.FRAM_ERR_USAGE
    with pytest.raises(fb.FramError):
        fb.fram_create(10, lam=-1.0)
    with pytest.raises(fb.FramError):
        fb.fram_create(10, schedule=fb.Schedule(theta=0.0))
    with pytest.raises(fb.FramError):
        fb.fram_create(10, schedule=fb.Schedule(alpha=1.5))
    with pytest.raises(fb.FramError):
        fb.fram_create(10, schedule=fb.Schedule(replay=[3, 0]))
    h = fb.fram_create(10, schedule=fb.Schedule(replay=[3, 4]))
    fb.fram_set_schedule(h, fb.Schedule(theta=2.0))
    del h


def test_sharded_create_validation():
    with pytest.raises(fb.FramError) as e:
        fb.fram_create_sharded(10, 1.0, None, b"\0" * 128, rank=0, world=3)
    assert e.value.status == fb.FRAM_ERR_USAGE


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np
    h = fb.fram_create(8)
    A = np.eye(8)
    with pytest.raises(fb.FramError) as e:
        fb.fram_solve(h, A, A)
    assert e.value.status == fb.FRAM_ERR_CUDA


def test_virtual_shard_validation():
    for n, w in ((10, 3), (16, 0), (16, 17)):
        with pytest.raises(fb.FramError) as e:
            fb.fram_create_sharded_virtual(n, 1.0, fb.Schedule(), world=w)
        assert e.value.status == fb.FRAM_ERR_USAGE


def test_replay_longer_than_max_outer_is_usage_error():
    # the stats trace arrays hold max_outer entries (include/fram.h): a longer replay is rejected up front
    with pytest.raises(fb.FramError) as e:
        fb.fram_create(16, schedule=fb.Schedule(max_outer=3, replay=[5, 5, 5, 5]))
    assert e.value.status == fb.FRAM_ERR_USAGE
    h = fb.fram_create(16, schedule=fb.Schedule(max_outer=4, replay=[5, 5, 5, 5]))
    assert h.schedule.max_outer == 4


def test_c_demo_no_cpu_fallback():
    # examples/fram_demo uses the C ABI from plain C with host buffers; without a GPU the solve must
    # fail with FRAM_ERR_CUDA (status 4), never fall back to a CPU computation
    import os
    import subprocess
    import torch
    from paper_2508_00887_b200 import build as b
    b.build()
    assert os.path.exists(b.DEMO_BIN)
    if torch.cuda.is_available():
        pytest.skip("a GPU is present: covered by test_gpu_c_demo")
    r = subprocess.run([b.DEMO_BIN, "32", "0"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 2 and "status 4" in r.stderr, (r.returncode, r.stderr)


@pytest.mark.gpu
@pytest.mark.parametrize("prec", [0, 2])
def test_gpu_c_demo(prec):
    # the same C program on the GPU: a noise-free relabelled weighted graph pair is matched exactly
    import subprocess
    from paper_2508_00887_b200 import build as b
    b.build()
    r = subprocess.run([b.DEMO_BIN, "64", str(prec)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, (r.stdout, r.stderr)
    assert "accuracy=1.0000" in r.stdout
