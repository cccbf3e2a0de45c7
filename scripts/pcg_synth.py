"""Per-iteration cost of the PRODUCT pcg_kernel<DIASYM7> on a synthetic operator.

    python scripts/pcg_synth.py [--n 10276240] [--variant 0]

Same size and diagonal offsets as config 4 (41 x 241 x 1040 logical grid), but
synthetic SPD coefficients, no remainder list, a random right-hand side and a
tolerance it cannot reach: two solves capped at K1 and K2 iterations give the
cost of one iteration as (T2 - T1) / (K2 - K1).  Beside scripts/iter_bench.cu
(the same loop as a stand-alone kernel) this tells whether the product kernel
loses time to its code or to the real operator's data.
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=10276240)
    ap.add_argument("--variant", type=int, default=0)
    ap.add_argument("--rem", type=int, default=0, help="1: an (empty) remainder list is attached")
    ap.add_argument("--tissue", type=int, default=0,
                    help="1: the TISSUE instantiation (b = M combo with M = A, no lift, no activation)")
    args = ap.parse_args()

    import torch

    from paper_2308_01651_b200 import _native as N
    from paper_2308_01651_b200.linalg import CgWorkspace

    n = args.n
    nx, nxy = 41, 41 * 241
    offs = [1, nx, nx + 1, nxy, nxy + 1, nxy + nx, nxy + nx + 1]
    ld = ((n + 31) // 32) * 32
    g = torch.Generator(device="cuda").manual_seed(1)
    vals = torch.zeros((1 + len(offs)) * ld, dtype=torch.float64, device="cuda")
    vals[:n] = 1.0 + 0.1 * torch.rand(n, generator=g, device="cuda", dtype=torch.float64)
    for s, d in enumerate(offs):
        v = -0.03 * torch.rand(n, generator=g, device="cuda", dtype=torch.float64)
        v[n - d:] = 0.0          # no coupling past the last row
        vals[(1 + s) * ld:(1 + s) * ld + n] = v
    dinv = 1.0 / vals[:n]
    b = torch.rand(n, generator=g, device="cuda", dtype=torch.float64)
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    ws = CgWorkspace(n)
    rem_ptr = torch.zeros((n + 31) // 32 + 1, dtype=torch.int32, device="cuda")
    rem_row = torch.zeros(1, dtype=torch.int32, device="cuda")

    def solve(max_iter):
        a = N.CgArgs()
        op = N.Operator()
        op.kind = N.OP_DIASYM
        op.n = n
        op.nnz = n * 15
        op.dia_np = len(offs)
        op.dia_ld = ld
        for s, d in enumerate(offs):
            op.dia_off[s] = d
        if args.rem:
            op.rem_n = 1
            op.rem_ptr = N.ptr(rem_ptr)
            op.rem_row = N.ptr(rem_row)
            op.rem_col = N.ptr(rem_row)
        a.op = op
        a.a_val = N.ptr(vals)
        a.dinv = N.ptr(dinv)
        a.b = N.ptr(b)
        if args.tissue:
            a.m_val = N.ptr(vals)
            a.combo = N.ptr(b)
            a.n_lift = 0
            a.dt = 1.0
        a.x = N.ptr(x)
        a.tol = 1e-300
        a.max_iter = max_iter
        a.variant = args.variant
        ws.status.zero_()
        ws.fill(a)
        x.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        N.check(N.lib().mdx_pcg_solve(N.C.byref(a), args.tissue, 0, N.stream_handle()),
                "mdx_pcg_solve")
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1), int(ws.iters.item()), float(ws.relres.item())

    solve(5)
    k1, k2 = 20, 100
    for _ in range(3):
        t1, i1, r1 = solve(k1)
        t2, i2, r2 = solve(k2)
        per = (t2 - t1) / (k2 - k1) * 1e3
        print(f"n={n} variant={args.variant} rem={args.rem} tissue={args.tissue}: {k1} it {t1:.3f} ms (iters {i1}, rel {r1:.2e}), "
              f"{k2} it {t2:.3f} ms (iters {i2}, rel {r2:.2e}) -> {per:.1f} us/iteration, "
              f"{160e-9 * n / (per * 1e-6):.0f} GB/s at 160 B")


if __name__ == "__main__":
    main()
