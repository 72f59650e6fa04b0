"""bench.py's launcher path on CPU (--dry-run, gloo): `--gpus N` without a launcher spawns N
ranks through torch.distributed.run, a torchrun launch at N = 1 and a plain run print the
same keys, the ranks' c3 shards tile the matrix in rank order, and --gpus must agree with
WORLD_SIZE."""

import json
import os
import socket
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "bench.py")


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(cmd, env=None):
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update(env or {})
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=300, env=e, cwd=ROOT)
    return p


def _line(p):
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout
    return json.loads(lines[0])


def test_plain_and_torchrun_lines_have_the_same_keys():
    plain = _line(_run([sys.executable, BENCH, "--dry-run"]))
    tr = _line(_run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
                     "--master-addr", "127.0.0.1", f"--master-port={_port()}", BENCH, "--gpus", "1", "--dry-run"]))
    assert set(plain) == set(tr)
    assert plain["n_gpus"] == tr["n_gpus"] == 1
    assert plain["dry_run"]["launcher"] == "direct" and tr["dry_run"]["launcher"] == "torch.distributed.run"
    assert plain["config"] == tr["config"]


def test_gpus_n_spawns_n_ranks():
    line = _line(_run([sys.executable, BENCH, "--gpus", "2", "--dry-run"]))
    assert line["n_gpus"] == 2 and line["dry_run"]["launcher"] == "torch.distributed.run"
    assert line["dry_run"]["shards"] == [[0, 79999], [80000, 159999]]
    assert line["config"]["q_total"] == 128


def test_gpus_must_match_world_size():
    p = _run([sys.executable, BENCH, "--gpus", "2", "--dry-run"], env={"WORLD_SIZE": "1"})
    assert p.returncode != 0 and "disagrees with WORLD_SIZE" in p.stderr
