"""Host-link bandwidth ceiling for the end-to-end (e2e) figures: pinned host -> device,
device -> host, and both directions at once (separate streams), 1 GiB buffers.

    python tools/micro/pcie_bw.py   (on a GPU box; prints one JSON line)
"""
import json

import torch


def main():
    n = 1 << 28                       # 1 GiB of f32
    dev = torch.device("cuda", 0)
    h_in = torch.empty(n, dtype=torch.float32).pin_memory()
    h_out = torch.empty(n, dtype=torch.float32).pin_memory()
    d_a = torch.empty(n, dtype=torch.float32, device=dev)
    d_b = torch.empty(n, dtype=torch.float32, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def timed(fn, reps=5):
        fn()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        torch.cuda.current_stream(dev).wait_stream(s1)
        torch.cuda.current_stream(dev).wait_stream(s2)
        e1.record()
        torch.cuda.synchronize(dev)
        return e0.elapsed_time(e1) / 1e3 / reps

    def h2d():
        with torch.cuda.stream(s1):
            d_a.copy_(h_in, non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            h_out.copy_(d_b, non_blocking=True)

    def both():
        h2d()
        d2h()
    b = n * 4
    t_h2d, t_d2h, t_both = timed(h2d), timed(d2h), timed(both)
    print(json.dumps({"h2d_gbs": round(b / t_h2d / 1e9, 2), "d2h_gbs": round(b / t_d2h / 1e9, 2),
                      "bidir_gbs_each": round(b / t_both / 1e9, 2), "bytes": b}))


if __name__ == "__main__":
    main()
