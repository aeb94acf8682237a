"""PCIe copy ceiling of the e2e leg: pinned host -> device and device -> pinned host over the
bench step's byte counts (170 MB in, 21 MB out), one direction at a time and both at once
(separate streams), CUDA events on the copy streams.  The e2e leg cannot beat H2D bytes / the
H2D rate measured here.

    python tools/pcie_peak.py
"""
import torch

H2D, D2H = 169869312, 20971520


def main():
    dev = torch.device("cuda:0")
    hi = torch.empty(H2D, dtype=torch.uint8, pin_memory=True)
    ho = torch.empty(D2H, dtype=torch.uint8, pin_memory=True)
    di = torch.empty(H2D, dtype=torch.uint8, device=dev)
    do = torch.empty(D2H, dtype=torch.uint8, device=dev)
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn, reps=10):
        best = None
        for _ in range(reps + 2):
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            torch.cuda.current_stream().wait_stream(s_in)
            torch.cuda.current_stream().wait_stream(s_out)
            b.record()
            b.synchronize()
            t = a.elapsed_time(b)
            best = t if best is None else min(best, t)
        return best

    def h2d():
        s_in.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s_in):
            di.copy_(hi, non_blocking=True)

    def d2h():
        s_out.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s_out):
            ho.copy_(do, non_blocking=True)

    def both():
        h2d()
        d2h()

    t_in, t_out, t_both = timed(h2d), timed(d2h), timed(both)
    print(f"H2D {H2D / 1e6:.1f} MB: {t_in:.3f} ms = {H2D / t_in / 1e6:.1f} GB/s")
    print(f"D2H {D2H / 1e6:.1f} MB: {t_out:.3f} ms = {D2H / t_out / 1e6:.1f} GB/s")
    print(f"both (two streams): {t_both:.3f} ms -> e2e ceiling {10.87e9 / (t_both * 1e-3) / 1e12:.2f} TF/s "
          f"for the 10.87 GFLOP step")


if __name__ == "__main__":
    main()
