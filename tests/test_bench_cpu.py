"""bench.py's multi-rank plumbing on the CPU: `--gpus 2` launches two ranks itself (torchrun, gloo in
--dry-run), they split the C3 domain into two slabs, the raw-sum all-gather covers every pixel once,
and rank 0 prints one JSON line with n_gpus = 2."""

import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_bench_spawns_ranks_dry_run():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--dry-run"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2
    assert line["slabs"] == [[0, 524288], [524288, 1048576]]


def test_bench_algorithmic_bytes():
    sys.path.insert(0, str(ROOT))
    import bench

    assert bench.bytes_per_vf(2, 4)["eval"] == 32 and bench.bytes_per_vf(3, 4)["eval"] == 44
    kb = bench.kernel_bytes_per_vf(2, 4)["algorithmic"]
    assert kb["k_ngf_sfeat2f"] + kb["k_ngf_adj4"] == 32 and kb["k_ngf_sfeat2"] == kb["k_ngf_sfeat2f"]
