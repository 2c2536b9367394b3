"""Background oracle sorts for the full-size parity tests (test infrastructure).

At BASELINE.json's full sizes the oracle (single-threaded mergesort,
oracle/oracle.c, the plain definition of) takes minutes per input.
The GPU test session starts these jobs as separate host processes as soon as
collection selects a full-size test, so they run on the host cores while the
other GPU tests run; each job regenerates its input from the seed
(synth_inputs, no method arithmetic), sorts it with the oracle and writes the
sorted bytes to a file.  The full-size tests then compare the GPU output with
that file element by element (oracle.parity).

Run one job by hand:  python tests/oracle_jobs.py NAME N SEED OUTFILE
"""
from __future__ import annotations

import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

DTYPE_OF = {"u64": 0, "f64": 1, "pair": 2, "rec100": 3, "u32": 4, "quartet": 5}

# (distribution, n, seed): every full-size input whose expected output is not
# already an exact closed form in test_gpu_fullsize.py.  Largest first.
FULLSIZE_JOBS = [
    ("uniform_u64", 1 << 30, 42),      # the headline bench.py times
    ("twodup_u64", 1 << 30, 3),        # c3
    ("zipf_u64", 1 << 30, 3),          # c3
    ("eightdup_u64", 1 << 30, 3),      # NEXT-2
    ("uniform_f64", 1 << 28, 2),       # c2
    ("exponential_f64", 1 << 28, 2),   # c2
    ("uniform_u32", 1 << 28, 6),       # NEXT-2
]
MAX_CONCURRENT = int(os.environ.get("IPS4O_ORACLE_JOBS", "7"))


def job_key(name: str, n: int, seed: int) -> str:
    return f"{name}_{n.bit_length() - 1}_{seed}"


def run_job(name: str, n: int, seed: int, out: str) -> None:
    sys.path.insert(0, ROOT)
    import oracle
    import synth_inputs as gen

    dt = DTYPE_OF[gen.DISTRIBUTIONS[name][0]]
    a = gen.generate(name, n, seed)
    t0 = time.time()
    oracle.sort_inplace(a, dt)
    dt_s = time.time() - t0
    tmp = out + ".part"
    a.tofile(tmp)
    os.replace(tmp, out)
    with open(out + ".time", "w") as f:
        f.write(f"{dt_s:.1f}\n")


class Pool:
    """Runs FULLSIZE_JOBS with at most MAX_CONCURRENT host processes."""

    def __init__(self, jobs=FULLSIZE_JOBS):
        self.dir = tempfile.mkdtemp(prefix="ips4o_oracle_")
        self.pending = list(jobs)
        self.running = {}
        self.done = {}
        self.failed = {}
        self._pump()

    def path(self, name, n, seed):
        return os.path.join(self.dir, job_key(name, n, seed) + ".bin")

    def _pump(self):
        for k, (p, job) in list(self.running.items()):
            rc = p.poll()
            if rc is None:
                continue
            del self.running[k]
            (self.done if rc == 0 else self.failed)[k] = job
        while self.pending and len(self.running) < MAX_CONCURRENT:
            job = self.pending.pop(0)
            name, n, seed = job
            p = subprocess.Popen([sys.executable, os.path.abspath(__file__), name, str(n), str(seed),
                                  self.path(name, n, seed)], cwd=ROOT)
            self.running[job_key(name, n, seed)] = (p, job)

    def wait(self, name, n, seed, timeout=3600.0):
        """Block until the job's output exists; return its path."""
        k = job_key(name, n, seed)
        t0 = time.time()
        while True:
            self._pump()
            if k in self.done:
                return self.path(name, n, seed)
            if k in self.failed:
                raise RuntimeError(f"oracle job {k} failed")
            if k not in self.running and all(job_key(*j) != k for j in self.pending):
                raise KeyError(f"no oracle job {k}")
            if time.time() - t0 > timeout:
                raise TimeoutError(f"oracle job {k} still running after {timeout} s")
            time.sleep(1.0)

    def close(self):
        for p, _ in self.running.values():
            p.kill()
        for f in os.listdir(self.dir):
            try:
                os.remove(os.path.join(self.dir, f))
            except OSError:
                pass
        try:
            os.rmdir(self.dir)
        except OSError:
            pass


if __name__ == "__main__":
    run_job(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4])
