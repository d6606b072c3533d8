"""Generate the committed golden fixtures from the reference itself.

Runs the reference's own C++ sources (oracle/_ref, compiled unmodified from
/root/reference/proj/src) on small seeded cases and stores inputs and
outputs as .npz: the ROM (build_rom), the dof map (index_global_nodes /
global_dof), the lifted load (assemble_global + lifting), the CG solution
(cg_solve, tol 1e-12, Jacobi) and the Gauss-point stresses
(evaluate_stress_in_element + von_mises). Run from the repo root:

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import refpy  # noqa: E402

CASES = {
    # name: (d, h, t, p, m_xy, m_z, q, rows, cols, kinds, delta_t, bc_mode)
    "tiny_mixed": (5e-6, 50e-6, 0.5e-6, 15e-6, 4, 3, 3, 2, 3, [0, 1, 0, 0, 0, 1],
                   [-250.0, -240.0, -260.0, -230.0, -270.0, -255.0], 1),
    "tiny_q4_literal": (4e-6, 40e-6, 0.4e-6, 10e-6, 6, 4, 4, 2, 2, None, [-250.0], 0),
    "tiny_clamped": (5e-6, 50e-6, 0.5e-6, 15e-6, 5, 4, 3, 1, 3, None, [-125.0], 2),
}


def main():
    for name, (d, h, t, p, mxy, mz, q, rows, cols, kinds, dts, bc) in CASES.items():
        r0 = refpy.build_rom(d, h, t, p, mxy, mz, q, 0, 71.7e9, 1)
        r1 = refpy.build_rom(d, h, t, p, mxy, mz, q, 1, 71.7e9, 1) if kinds is not None else None
        k = None if kinds is None else np.array(kinds, np.uint8)
        s = refpy.RefSession(r0, r1, rows, cols, kinds=k, delta_t=np.array(dts), bc_mode=bc)
        b, cm, _ = s.rhs()
        u, it, rr = s.iterate(1e-12, 10000, 1, 1)
        stress = s.recover(u, 8, threads=1)
        out = dict(geometry=np.array([d, h, t, p]), mesh=np.array([mxy, mz, q]), rows=rows, cols=cols,
                   kinds=np.zeros(0, np.uint8) if k is None else k, delta_t=np.array(dts), bc_mode=bc,
                   dof_map=s.dof_map(), load=b, constrained=cm, u=u, iterations=it, relres=rr, stress=stress)
        for tag, r in (("tsv", r0), ("dummy", r1)):
            if r is None:
                continue
            out.update({f"{tag}_K": r.K, f"{tag}_b_el": r.b_el, f"{tag}_Phi": r.Phi, f"{tag}_u_T": r.u_T,
                        f"{tag}_gx": r.gx, f"{tag}_gy": r.gy, f"{tag}_gz": r.gz, f"{tag}_elem_mat": r.elem_mat,
                        f"{tag}_mats": r.mats, f"{tag}_fingerprint": np.frombuffer(r.fingerprint, np.uint8)})
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **out)
        print(f"{name}: N={s.N} iterations={it} -> {os.path.relpath(path)} ({os.path.getsize(path)} B)")


if __name__ == "__main__":
    main()
