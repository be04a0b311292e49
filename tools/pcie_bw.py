"""Pinned host <-> device copy bandwidth on this box: H2D alone, D2H alone, both at once on two
streams (the full-duplex bound of the e2e leg of bench.py).  python tools/pcie_bw.py [MB]"""
import sys
import time

import torch


def main():
    mb = int(sys.argv[1]) if len(sys.argv) > 1 else 175
    n = mb * (1 << 20) // 4
    h_src = torch.empty(n, dtype=torch.float32).pin_memory()
    h_dst = torch.empty(n, dtype=torch.float32).pin_memory()
    d_a = torch.empty(n, dtype=torch.float32, device="cuda")
    d_b = torch.empty(n, dtype=torch.float32, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn, reps=10):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / reps

    def h2d():
        with torch.cuda.stream(s1):
            d_a.copy_(h_src, non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            h_dst.copy_(d_b, non_blocking=True)

    def both():
        h2d()
        d2h()

    nb = n * 4
    t1, t2, t3 = timed(h2d), timed(d2h), timed(both)
    print(f"{mb} MB: H2D {nb / t1 / 1e9:.1f} GB/s ({t1 * 1e3:.2f} ms), D2H {nb / t2 / 1e9:.1f} GB/s "
          f"({t2 * 1e3:.2f} ms), both concurrently {t3 * 1e3:.2f} ms ({2 * nb / t3 / 1e9:.1f} GB/s total)")


if __name__ == "__main__":
    main()
