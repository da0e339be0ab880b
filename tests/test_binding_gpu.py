"""The Python binding validates every caller-supplied buffer and plan before
calling into libtsm (the C ABI cannot see buffer sizes, so a wrong
`out`, plan or second operand would become an out-of-bounds device access)."""
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tsm():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_1905_03136_b200 import binding
    return binding


def _t(*shape, dt=torch.float64):
    return torch.zeros(*shape, dtype=dt, device="cuda")


def test_tsmttsm_rejects_bad_out_and_plan(tsm):
    A, B = _t(100, 8), _t(100, 4)
    with pytest.raises(ValueError, match="shape"):
        tsm.tsmttsm(A, B, out=_t(8, 3))
    with pytest.raises(ValueError, match="dtype"):
        tsm.tsmttsm(A, B, out=_t(8, 4, dt=torch.complex128))
    with pytest.raises(ValueError, match="plan"):
        tsm.tsmttsm(A, B, plan=tsm.get_plan("tsmttsm", "d", 8, 8, 0))
    with pytest.raises(ValueError, match="plan"):
        tsm.tsmttsm(A, B, plan=tsm.get_plan("tsmm", "d", 8, 4, 0))
    with pytest.raises(ValueError):
        tsm.tsmttsm(A, _t(99, 4))
    with pytest.raises(ValueError):
        tsm.tsmttsm(A, _t(100, 4, dt=torch.complex128))
    with pytest.raises(ValueError, match="conj"):
        tsm.tsmttsm(A.to(torch.complex128), B.to(torch.complex128),
                    plan=tsm.get_plan("tsmttsm", "z", 8, 4, 0), conj=True)
    C = tsm.tsmttsm(A, B, out=_t(8, 4))  # the right buffer still works
    assert C.shape == (8, 4)


def test_tsmm_rejects_bad_out_and_plan(tsm):
    A, C = _t(100, 8), _t(8, 5)
    with pytest.raises(ValueError, match="shape"):
        tsm.tsmm(A, C, out=_t(99, 5))
    with pytest.raises(ValueError, match="shape"):
        tsm.tsmm(A, C, out=_t(100, 6))
    with pytest.raises(ValueError, match="dtype"):
        tsm.tsmm(A, C, out=_t(100, 5, dt=torch.complex128))
    with pytest.raises(ValueError, match="plan"):
        tsm.tsmm(A, C, plan=tsm.get_plan("tsmm", "d", 8, 8, 0))
    with pytest.raises(ValueError):
        tsm.tsmm(A, _t(7, 5))
    with pytest.raises(ValueError):
        tsm.tsmm(A, _t(8, 5, dt=torch.complex128))


def test_update_and_cgs_reject_mismatches(tsm):
    A, C, B = _t(100, 8), _t(8, 5), _t(100, 5)
    with pytest.raises(ValueError):
        tsm.tsmm_update(A, C, _t(99, 5), -1.0, 1.0)
    with pytest.raises(ValueError, match="plan"):
        tsm.tsmm_update(A, C, B, -1.0, 1.0, plan=tsm.get_plan("tsmm", "d", 8, 6, 0))
    with pytest.raises(ValueError):
        tsm.cgs_step(A, _t(99, 5))
    with pytest.raises(ValueError, match="C"):
        tsm.cgs_step(A, B, C=_t(5, 8))
    with pytest.raises(ValueError, match="plan"):
        tsm.cgs_step(A, B, p_tt=tsm.get_plan("tsmttsm", "d", 8, 8, 0))
    with pytest.raises(ValueError, match="plan"):
        tsm.cgs_step(A, B, p_mm=tsm.get_plan("tsmttsm", "d", 8, 5, 0))


def test_shared_kernel_smem_attribute_only_grows():
    """Plans with the same kernel function but different run-time stages share
    the function's max-dynamic-shared-memory attribute: a later plan with
    fewer stages must not lower it under an earlier plan (GPU suite run 12:
    'cudaLaunchKernel: invalid argument' on the earlier plan)."""
    import numpy as np
    import oracle
    import tsminputs as ti
    from paper_1905_03136_b200 import binding as tsm
    cfg = dict(threads=288, rows_per_chunk=64, p0=2, p1=2, p2=24, p3=24, stages=6, ctas_per_sm=1, kernel=1, p3_=0)
    cfg.pop("p3_")
    big = tsm.Plan("tsmttsm", "d", 24, 24, 0, config=cfg)
    small = tsm.Plan("tsmttsm", "d", 24, 24, 0, config=dict(cfg, stages=2))
    assert big.config()["stages"] > small.config()["stages"]
    A = ti.matrix(100003, 24, "A")
    B = ti.matrix(100003, 24, "B")
    for plan in (big, small, big):
        got = tsm.tsmttsm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), plan=plan).cpu().numpy()
        ref, bound = oracle.tsmttsm(A, B)
        assert oracle.max_err_ratio(got, ref, bound)[0] <= 1e-12
    assert np.isfinite(got).all()
