import os
import subprocess
import sys
import tempfile
import time

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HERE = os.path.dirname(os.path.abspath(__file__))
for _p in (ROOT, HERE):
    if _p not in sys.path:
        sys.path.insert(0, _p)

FULLRUN_MODULE = "test_fullrun_gpu.py"
_JOBS = {}   # name -> (Popen, out path, log path)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through the C ABI)")
    config.addinivalue_line("markers", "slow: long CPU test")


def _fullrun_names(item):
    return [m.args[0] for m in item.iter_markers("oracle_run")]


@pytest.hookimpl(trylast=True)   # after -m / -k deselection: start only the jobs of selected tests
def pytest_collection_modifyitems(session, config, items):
    """The full-length parity tests (test_fullrun_gpu.py) go last, and their serial fp64 oracle
    runs start now, each in its own process (tests/oracle_job.py), so they overlap every other
    test instead of running one after another."""
    late = [it for it in items if it.fspath.basename == FULLRUN_MODULE]
    if not late:
        return
    items[:] = [it for it in items if it.fspath.basename != FULLRUN_MODULE] + late
    names = sorted({n for it in late for n in _fullrun_names(it)})
    tmp = tempfile.mkdtemp(prefix="zpic_oracle_jobs_")
    for name in names:
        out = os.path.join(tmp, name + ".npz")
        log = open(os.path.join(tmp, name + ".log"), "w")
        proc = subprocess.Popen([sys.executable, os.path.join(HERE, "oracle_job.py"), name, out],
                                stdout=log, stderr=subprocess.STDOUT, cwd=ROOT)
        _JOBS[name] = (proc, out, log.name)


def pytest_unconfigure(config):
    for proc, _, _ in _JOBS.values():
        if proc.poll() is None:
            proc.kill()


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.build()
    return oracle


@pytest.fixture
def oracle_run(request):
    """The background oracle run(s) named by the test's @pytest.mark.oracle_run(name): waits for
    the process and returns its npz contents (a dict)."""
    def get(name, timeout=3600):
        if name not in _JOBS:   # the test was selected by itself: run the job now
            out = os.path.join(tempfile.mkdtemp(prefix="zpic_oracle_job_"), name + ".npz")
            subprocess.check_call([sys.executable, os.path.join(HERE, "oracle_job.py"), name, out], cwd=ROOT)
            return dict(np.load(out))
        proc, out, log = _JOBS[name]
        t0 = time.time()
        while proc.poll() is None:
            if time.time() - t0 > timeout:
                proc.kill()
                raise TimeoutError("oracle job %s" % name)
            time.sleep(1.0)
        if proc.returncode != 0:
            raise RuntimeError("oracle job %s failed:\n%s" % (name, open(log).read()[-4000:]))
        return dict(np.load(out))
    return get
