"""bench.py's N > 1 launch contract, on CPU (no GPU needed): a torchrun world that does not match
--gpus is refused (exit 2) before any device work, so a scaling run can never silently measure
fewer ranks than it claims."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_world_size_must_match_gpus():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "1", "--steps", "1"],
                       env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 2
    assert "WORLD_SIZE=2 but --gpus 1" in r.stderr


def test_r_alg_bytes_follow_survey_8d():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.r_alg_bytes(64, 1) == 11
    assert bench.r_alg_bytes(100, 1) == 16
    assert bench.r_alg_bytes(300, 1) == 44
    assert bench.r_alg_bytes(2000, 2) == 20
