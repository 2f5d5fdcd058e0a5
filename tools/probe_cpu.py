"""host LAPACK scaling on the GPU box (profiling aid): batched 48x48 SVDs with a
thread pool vs a process pool"""
import os
import time
from concurrent.futures import ProcessPoolExecutor, ThreadPoolExecutor

import numpy as np
from threadpoolctl import threadpool_limits

a = np.random.default_rng(0).standard_normal((4000, 48, 48))


def work(chunk):
    with threadpool_limits(1):
        return np.linalg.svd(chunk, full_matrices=False)[1].sum()


if __name__ == "__main__":
    n = os.cpu_count()
    t = time.time(); work(a); t1 = time.time() - t
    parts = np.array_split(a, n)
    with ThreadPoolExecutor(n) as ex:
        t = time.time(); list(ex.map(work, parts)); tt = time.time() - t
    with ProcessPoolExecutor(n) as ex:
        list(ex.map(work, parts))
        t = time.time(); list(ex.map(work, parts)); tp = time.time() - t
    print(f"cpus {n}: 4000 x 48x48 svd: serial {t1:.2f}s, {n} threads {tt:.2f}s, {n} processes {tp:.2f}s")
