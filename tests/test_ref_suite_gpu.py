"""The reference's OWN test files, unchanged, against the B200 engine.

tests/ref_suite/gsetbench_b200.py leaves the unmodified reference package
(staged under baseline/_ref by __graft_entry__.build(); never committed) in
place and rebinds its run_trial / run_campaign to this repo's engine -- the
executable form of INTEGRATION.md's reference-side binding.  The reference's
pytest files are then run from baseline/_ref/pkg/tests in a subprocess with
that binding loaded as a pytest plugin (-p gsetbench_b200), so drop-in
compatibility is asserted by the reference's suite
(pkg/tests/test_solvers.py:18-101, test_campaign.py:159-254,
test_acceptance.py:255-317), not by a restatement of it.
"""

import os
import re
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

REF_TESTS = ROOT / "baseline" / "_ref" / "pkg" / "tests"
BIND = ROOT / "tests" / "ref_suite"
REF_SRC = ROOT / "baseline" / "_ref" / "pkg" / "src"


def _run(files, extra=()):
    if not (REF_TESTS / "test_solvers.py").exists():
        pytest.skip("reference tests not staged (baseline/_ref is made by __graft_entry__.build() "
                    "in the build container)")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([str(BIND), str(REF_SRC), str(ROOT)]))
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-p", "gsetbench_b200",
           "--rootdir", str(REF_TESTS), *extra, *[str(REF_TESTS / f) for f in files]]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, cwd=REF_TESTS, env=env)
    tail = (out.stdout + out.stderr)[-3000:]
    assert out.returncode == 0, tail
    m = re.search(r"(\d+) passed", out.stdout)
    assert m, tail
    return int(m.group(1)), out.stdout


def test_shim_binds_the_engine():
    """The shim's run_trial is the GPU engine's and equals the unmodified
    reference's run_trial on the same instance and seed."""
    code = (
        "import gsetbench_b200, gsetbench.solvers as s, gsetbench.campaign as c\n"
        "assert s.run_trial.__module__ == 'gsetbench_b200' and c.run_trial is s.run_trial\n"
        "from gsetbench.instances import TorusSpec, generate_torus\n"
        "inst = generate_torus(TorusSpec(6, 8, 3))\n"
        "r = s.run_trial(inst, s.default_config(s.ANNEALING, 40, 11))\n"
                "print(r.best_cut, r.sweeps_executed, ''.join('1' if x > 0 else '0' for x in r.best_spins))\n")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([str(BIND), str(REF_SRC), str(ROOT)]))
    if not (REF_TESTS / "test_solvers.py").exists():
        pytest.skip("reference not staged")
    ours = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                          timeout=600, env=env)
    assert ours.returncode == 0, ours.stderr[-2000:]
    plain = code.replace("import gsetbench_b200, ", "import ").replace(
        "assert s.run_trial.__module__ == 'gsetbench_b200' and c.run_trial is s.run_trial\n",
        "assert s.run_trial.__module__ == 'gsetbench.solvers'\n")
    env_ref = dict(os.environ, PYTHONPATH=str(REF_SRC))
    ref = subprocess.run([sys.executable, "-c", plain], capture_output=True, text=True,
                         timeout=600, env=env_ref)
    assert ref.returncode == 0, ref.stderr[-2000:]
    assert ours.stdout == ref.stdout and ours.stdout.strip()


def test_reference_solver_campaign_acceptance_suites_pass_on_the_engine():
    n, _ = _run(["test_solvers.py", "test_campaign.py", "test_acceptance.py"])
    assert n >= 40


def test_rest_of_the_reference_suite_still_passes_through_the_shim():
    """The files off the sweep path (codec, evaluate, instances, metrics, oracle,
    registry) are the reference's own modules; the CLI's solve / campaign /
    report commands run their trials on the engine."""
    n, _ = _run(["test_codec.py", "test_evaluate.py", "test_instances.py", "test_metrics.py",
                 "test_oracle.py", "test_registry.py", "test_cli.py"])
    assert n >= 60
