"""Observed rounding error of the Rock4 forced step on a Neumann eigenmode (GPU) against R_s(z) v,
in units of eps_mach * s * max|w| (the bound used by tests/test_gpu_mr_rock4.py::test_rock4_forced_eigenmode)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_04651_b200 as P  # noqa: E402


def main():
    J, n = 7, 128
    k1, k2 = 3, 5
    xx = (np.arange(n) + 0.5) / n
    v = np.outer(np.cos(np.pi * k2 * xx), np.cos(np.pi * k1 * xx))
    u = torch.tensor(v[None], device="cuda").reshape(1, -1)
    g = P.Grid.build(2, J, J, 0.0, P.mr_rowmajor_to_morton(2, J, u))
    _, vm = g.leaf_tensors()
    vm = vm.cpu().numpy()
    eps = 2.5e-3
    lam = -eps * 4 * n * n * (np.sin(np.pi * k1 / (2 * n)) ** 2 + np.sin(np.pi * k2 / (2 * n)) ** 2)
    for mode in ("mat", "free"):
        os.environ["RDMR_R4_MODE"] = mode
        for s in (5, 7, 12, 25, 40):
            c = P.rock4_coeffs(s)
            for frac in (0.5, 0.9):
                h = frac * c["ell"] / (eps * g.info()["rho1"])
                out, err = g.rock4_forced_step(torch.tensor(vm[0], device="cuda"), eps, h, s)
                z = h * lam
                Pm, Pc = 0.0, 1.0
                for mu, nu, ka in zip(c["mu"], c["nu"], c["kappa"]):
                    Pm, Pc = Pc, (nu + mu * z) * Pc + ka * Pm
                sg = c["sigma"]
                R = (1 + z * (sg[0] + z * (sg[1] + z * (sg[2] + z * sg[3])))) * Pc
                zz = -np.linspace(0, c["ell"], 4001)
                wmax = np.abs(1 + zz * (sg[0] + zz * (sg[1] + zz * (sg[2] + zz * sg[3])))).max()
                e1 = np.max(np.abs(out.cpu().numpy() - R * vm[0]))
                e2 = np.max(np.abs(err.cpu().numpy() - sg[3] * z ** 4 * Pc * vm[0]))
                unit = np.finfo(float).eps * s * wmax
                print(f"{mode} s={s:3d} h/hmax={frac} wmax={wmax:.2e} out_err={e1:.2e} ({e1/unit:.3f} u) "
                      f"est_err={e2:.2e} ({e2/unit:.3f} u)  s^2*1e-12={1e-12*s*s:.1e}")


if __name__ == "__main__":
    main()
