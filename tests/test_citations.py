"""Every `file.py:N` citation of the reference in this repository points inside the cited
file, and the anchors the boundary and the oracle lean on name the right definitions.

The line counts below are the reference's (kaczbench at /root/reference/pkg, PAPER.md,
SPEC.md); the anchor check reads the reference itself when it is present (the build
container), so the table cannot drift from the files it describes."""

import glob
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference"

REF_LINES = {"__init__.py": 75, "cgls.py": 91, "cli.py": 220, "distributed.py": 363, "errors.py": 58,
             "harness.py": 225, "linalg.py": 88, "parallel.py": 368, "reports.py": 161, "sampling.py": 131,
             "solvers.py": 371, "spectral.py": 156, "sysgen.py": 271, "conftest.py": 38,
             "test_acceptance.py": 275, "test_cli.py": 100, "test_distributed.py": 173, "test_harness.py": 156,
             "test_linalg.py": 111, "test_parallel.py": 139, "test_sampling.py": 118, "test_solvers_seq.py": 248,
             "test_spectral.py": 122, "test_sysgen.py": 161, "PAPER.md": 556, "SPEC.md": 645}

# (file, line, text the line must contain) -- the definitions include/kz_b200.h, oracle/ and the
# package docstrings cite most
ANCHORS = [
    ("sampling.py", 34, "class Prng"), ("sampling.py", 47, "SeedSequence"), ("sampling.py", 67, "def worker_rng"),
    ("sampling.py", 89, "def sample"), ("sampling.py", 91, "searchsorted"), ("sampling.py", 101, "def make_sampler"),
    ("sampling.py", 107, "EmptyRangeError"), ("sampling.py", 108, "np.cumsum"), ("sampling.py", 109, "cdf[-1]"),
    ("sampling.py", 119, "def partition_bounds"), ("linalg.py", 80, "def row_norm_cache"),
    ("linalg.py", 83, "einsum"), ("solvers.py", 107, "def kaczmarz_step"), ("solvers.py", 120, "def rka_combined_step"),
    ("solvers.py", 140, "def rkab_worker_block"), ("solvers.py", 148, "def resolve_alphas"),
    ("solvers.py", 162, "def worker_streams"), ("solvers.py", 174, "def _trace_record"), ("solvers.py", 182, "def _drive"),
    ("solvers.py", 271, "def solve_ck"), ("solvers.py", 294, "def solve_rk"), ("solvers.py", 313, "def solve_rka_seq"),
    ("solvers.py", 337, "def solve_rkab_seq"), ("harness.py", 72, "def _run_cgls"), ("harness.py", 98, "def run_solver"),
    ("harness.py", 127, "def measure_iterations"), ("harness.py", 160, "def timed_replay"),
    ("harness.py", 180, "def trace_run"), ("harness.py", 199, "def bench"), ("parallel.py", 175, "def solve_rka_parallel"),
    ("parallel.py", 221, "q * sqn[i]"), ("distributed.py", 119, "def allreduce_sum"),
    ("distributed.py", 204, "def make_partition"), ("distributed.py", 282, "def solve_rka_dist"),
    ("distributed.py", 339, "def run_distributed_solve"), ("cgls.py", 18, "def _cgls_pass"),
    ("cgls.py", 42, "def cgls_solve"), ("spectral.py", 66, "def spectral_stats"), ("spectral.py", 124, "def optimal_alpha"),
    ("spectral.py", 137, "def partial_alphas"), ("sysgen.py", 125, "def generate_mother"),
    ("sysgen.py", 190, "def save_system"),
]

CITE = re.compile(r"(?<![\w/])(?:kaczbench/)?([a-z_]+\.py|PAPER\.md|SPEC\.md):(\d+)(?:-(\d+))?")
# files written by the survey / judge / advisor, not by this repository's code
SKIP = {"SURVEY.md", "BASELINE.md", "VERDICT.md", "ADVICE.md", "PAPERS.md", "SNIPPETS.md"}


def _repo_files():
    for f in glob.glob(os.path.join(ROOT, "**", "*"), recursive=True):
        rel = os.path.relpath(f, ROOT)
        if not os.path.isfile(f) or rel in SKIP or rel.startswith(("gpurun_out", ".git", "wt_", "baseline")):
            continue
        if rel.rsplit(".", 1)[-1] in ("py", "c", "h", "cu", "cuh", "md", "sh"):
            yield rel


def test_every_reference_citation_is_in_range():
    bad = []
    for rel in _repo_files():
        with open(os.path.join(ROOT, rel), errors="ignore") as fh:
            for ln, line in enumerate(fh, 1):
                for m in CITE.finditer(line):
                    name = m.group(1)
                    if name not in REF_LINES:
                        continue
                    a = int(m.group(2))
                    b = int(m.group(3) or a)
                    if not (1 <= a <= b <= REF_LINES[name]):
                        bad.append(f"{rel}:{ln}: {m.group(0)} (file has {REF_LINES[name]} lines)")
    assert not bad, "\n".join(bad)


@pytest.mark.skipif(not os.path.isdir(REF), reason="the reference is only present in the build container")
def test_reference_line_counts_and_anchors():
    src = os.path.join(REF, "pkg", "src", "kaczbench")
    for name, n in REF_LINES.items():
        for d in (src, os.path.join(REF, "pkg", "tests"), REF):
            p = os.path.join(d, name)
            if os.path.isfile(p):
                with open(p) as fh:
                    assert sum(1 for _ in fh) == n, name
                break
    for name, line, text in ANCHORS:
        with open(os.path.join(src, name)) as fh:
            lines = fh.readlines()
        assert text in lines[line - 1], (name, line, lines[line - 1])
