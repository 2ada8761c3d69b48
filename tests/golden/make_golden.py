"""Generate the golden fixtures from the UNMODIFIED reference (oracle/_ref).

Run here (where /root/reference exists):  python tests/golden/make_golden.py
The fixtures pin the oracle restatement (tests/test_oracle.py) and the GPU path
(tests/test_golden_gpu.py) on machines where the reference sources are absent.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import ref  # noqa: E402

sys.path.insert(0, os.path.dirname(HERE))
from fieldsets import custom_fields  # noqa: E402


def case(name, family, d, order, dt, T, dt_leb, M, seed, rec, em_dt, fields=None, kappas=(0, 2)):
    ops = ref.Ops(family, d, order=order, fields=fields)
    values, _ = ref.simulate_brownian(T, dt_leb, M, seed)
    phi = ops.datum()
    ms, mst, _ = ops.solve_magnus(values, dt_leb, T, dt, record_times=rec, seed=seed)
    es, est, _ = ops.solve_euler(values, dt_leb, T, em_dt, record_times=rec, seed=seed)
    out = dict(family=family, d=d, order=order, dt=dt, T=T, dt_leb=dt_leb, M=M, seed=seed,
               record_times=np.asarray(rec, float), em_dt=em_dt, values=values, phi=phi,
               magnus=ms, magnus_status=mst, euler=es, euler_status=est)
    # window-0 trace of path 0: functionals, union fill, one_norm, expmv report
    f5 = ref.functionals(values[0], 0, int(round(dt / dt_leb)), dt_leb)
    rp, ci, v = ops.fill(order, f5)
    y, rep = ref.expmv(rp, ci, v, phi)
    out.update(trace_f5=f5, trace_norm=ref.one_norm(rp, ci, v), trace_y=y,
               trace_segments=rep["segments"], trace_max_terms=rep["max_terms"],
               trace_nnz=len(v))
    for s, slot in enumerate(ref.SLOTS):
        c = ops.csr(slot)
        if c is not None:
            out[f"csr_{slot}_rp"], out[f"csr_{slot}_ci"], out[f"csr_{slot}_v"] = c
    for k in ref.FIELD_NAMES:
        a, zero = ops.field(k)
        if not zero:
            out[f"field_{k}"] = a
    if family == "langevin-constant":
        ex = ops.exact_reference(values, dt_leb, T, seed=seed)
        out["exact"] = ex
        for kappa in kappas:
            e = ops.errors(kappa, ex, ms[-1], app_status=mst[-1], seed=seed)
            out[f"err_k{kappa}"] = np.array([e["err"], e["ame"], e["blowups"], e["excluded"]])
            out[f"me_k{kappa}"] = e["me"]
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, "magnus status", mst[-1], "euler status", est[-1])


if __name__ == "__main__":
    # cfg1 shape (64x64, constant, order 2), shortened horizon
    case("cfg1_const64_o2", "langevin-constant", 64, 2, 0.1, 0.2, 1e-4, 3, 424242, [0.1], 1e-4)
    case("var20_o3", "langevin-variable", 20, 3, 0.05, 0.1, 1e-3, 3, 1, [0.05], 1e-3)
    case("custom12_o3", "fields", 12, 3, 0.05, 0.1, 1e-3, 2, 5, [], 1e-3, fields=custom_fields(12))
    case("const16_o3_blowcap", "langevin-constant", 16, 3, 0.1, 0.2, 1e-3, 2, 9, [0.1], 1e-3)
