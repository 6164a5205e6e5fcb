"""PCIe duplex probe: pinned H2D and D2H copy times alone and concurrently
(separate streams), for the e2e floor analysis of the host entry point
(DESIGN.md 7 "e2e").  Prints one JSON line."""
import json
import time

import torch


def main():
    dev = torch.device("cuda:0")
    n_in, n_out = 132 << 20, 268 << 20
    h_in = torch.empty(n_in, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(n_out, dtype=torch.uint8).pin_memory()
    d_in = torch.empty(n_in, dtype=torch.uint8, device=dev)
    d_out = torch.empty(n_out, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def t(fn, reps=5):
        best = 1e9
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        return best * 1e3

    def h2d():
        with torch.cuda.stream(s1):
            d_in.copy_(h_in, non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)

    def both():
        h2d()
        d2h()

    a, b, c = t(h2d), t(d2h), t(both)
    print(json.dumps({"h2d_132MiB_ms": a, "d2h_268MiB_ms": b, "concurrent_ms": c,
                      "h2d_GBs": n_in / a / 1e6, "d2h_GBs": n_out / b / 1e6,
                      "duplex_efficiency": max(a, b) / c}))


if __name__ == "__main__":
    main()
