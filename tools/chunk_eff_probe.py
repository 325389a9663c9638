"""Device time of the K1 pass over the first n DAGs of the C5 corpus (Session,
one stream) for several n: how much a chunked pass loses per DAG."""
import statistics
import sys

sys.path.insert(0, ".")
from paper_2602_20826_b200 import _lib  # noqa: E402

corpus = _lib.Corpus(1000000, pinned=True, seed=1, gpu=True)
b = corpus.batch()
for n in (62500, 125000, 200000, 250000, 333334, 500000, 1000000):
    s = _lib.Session(b.slice(0, n), 148)
    for _ in range(3):
        s.run()
    ms = statistics.median(s.run() for _ in range(15))
    kt = s.kernel_times()
    print(f"n {n:8d}  {ms:.3f} ms  {1e6 * ms / n:.2f} ns/DAG  " +
          "  ".join(f"{k} {v:.3f}" for k, v in kt.items()), flush=True)
