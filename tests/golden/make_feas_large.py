"""Generate tests/golden/feas_large.json: fleet feasibility and canonical partitions of random
slice vectors at n = 16, 32, 64 from the REFERENCE itself (reference mig.py:144-181,
MigTopology.partition_fleet), each query under a per-query time limit (the reference's memoised
backtracking can take seconds on infeasible vectors; timed-out queries are dropped and counted).

Vectors, alternately: (a) the slice multiset of n random table rows, then 0-3 random
single-slice edits (add, remove or change one slice); (b) slice counts drawn directly with
total compute units in [6n, 7n + 1], so packing limits (one 4g or 7g per GPU, two 3g) decide.
Run here (the reference is importable in this container only):
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_feas_large.py [count_per_n]
"""
import json
import os
import random
import signal
import sys
import time

from carbon_sched.core import SLICE_ORDER
from carbon_sched.mig import _build_default_topology

COUNT = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
LIMIT_S = 1.0


class Timeout(Exception):
    pass


def _alarm(signum, frame):
    raise Timeout()


def main():
    signal.signal(signal.SIGALRM, _alarm)
    rng = random.Random(2304_09781)
    out = {"source": "reference carbon_sched.mig.MigTopology.partition_fleet (mig.py:144-181)",
           "slice_order": [s.label for s in SLICE_ORDER], "limit_s": LIMIT_S, "cases": [], "timeouts": {}}
    for n in (16, 32, 64):
        topo = _build_default_topology()
        rows = [(cid, [sum(1 for s in topo.config_slices(cid) if s == t) for t in SLICE_ORDER]) for cid in topo.config_ids]
        t0, done, timeouts = time.time(), 0, 0
        while done < COUNT:
            if done % 2:
                # direct counts near the capacity boundary: total compute units in [6n, 7n + 1]
                while True:
                    a = rng.randrange(n // 4 + 1)
                    b = rng.randrange(n - a + 1)
                    c = rng.randrange(2 * (n - a) + 1)
                    d = rng.randrange(3 * (n - a) + 1)
                    rest = 7 * n + rng.randrange(-n, 2) - (7 * a + 4 * b + 3 * c + 2 * d)
                    if rest >= 0:
                        vec = [a, b, c, d, rest]
                        break
                slices = [t for t, cnt in zip(SLICE_ORDER, vec) for _ in range(cnt)]
                signal.setitimer(signal.ITIMER_REAL, LIMIT_S)
                try:
                    part = topo.partition_fleet(slices, n)
                except Timeout:
                    timeouts += 1
                    topo = _build_default_topology()
                    continue
                finally:
                    signal.setitimer(signal.ITIMER_REAL, 0)
                out["cases"].append([n] + vec + [list(part) if part is not None else None])
                done += 1
                continue
            vec = [0] * 5
            for _ in range(n):
                _cid, r = rows[rng.randrange(len(rows))]
                vec = [a + b for a, b in zip(vec, r)]
            for _ in range(rng.randrange(4)):
                k = rng.randrange(5)
                op = rng.randrange(3)
                if op == 0:
                    vec[k] += 1
                elif op == 1 and vec[k] > 0:
                    vec[k] -= 1
                else:
                    j = rng.randrange(5)
                    if vec[k] > 0:
                        vec[k] -= 1
                        vec[j] += 1
            slices = [t for t, c in zip(SLICE_ORDER, vec) for _ in range(c)]
            signal.setitimer(signal.ITIMER_REAL, LIMIT_S)
            try:
                part = topo.partition_fleet(slices, n)
            except Timeout:
                timeouts += 1
                topo = _build_default_topology()   # drop a cache left mid-search
                continue
            finally:
                signal.setitimer(signal.ITIMER_REAL, 0)
            out["cases"].append([n] + vec + [list(part) if part is not None else None])
            done += 1
        out["timeouts"][str(n)] = timeouts
        print("n=%d: %d cases, %d timeouts, %.1f s" % (n, done, timeouts, time.time() - t0), file=sys.stderr)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "feas_large.json")
    with open(path, "w") as fh:
        json.dump(out, fh, separators=(",", ":"))


if __name__ == "__main__":
    main()
