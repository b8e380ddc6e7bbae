"""tfla_train_step_host: one forward + backward with HOST buffers (the
reference's host-tensor boundary, chunkwise.hpp:39-54), streamed in batch-row
slices through device slots on three streams. Its outputs are bit-identical to
the device-buffer entry points called on the same batch rows."""
import numpy as np
import pytest

from tests._util import make_case


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("shape", [(3, 2, 256, 64, 64, 64), (5, 1, 512, 128, 256, 256)])
def test_host_step_matches_device_path(variant, shape):
    import torch

    from paper_2503_14376_b200 import (Dims, SequenceInputs, Variant, chunkwise_backward, chunkwise_forward,
                                       train_step_host)

    B, H, T, L, dqk, dhv = shape
    q, k, v, ip, fp = make_case(B, H, T, dqk, dhv, seed=41 + variant)
    rng = np.random.default_rng(42)
    bf = lambda a: torch.from_numpy(np.asarray(a, dtype=np.float32)).to(torch.bfloat16).contiguous().pin_memory()
    f32 = lambda a: torch.from_numpy(np.asarray(a, dtype=np.float32)).contiguous().pin_memory()
    host = SequenceInputs(bf(q), bf(k), bf(v), f32(ip), f32(fp))
    dh = bf(rng.standard_normal((B, H, T, dhv)))
    dims = Dims(T=T, L=L, d_qk=dqk, d_hv=dhv, n_head=H, n_batch=B)
    for rep in range(2):  # second call reuses the cached device slots
        h, g = train_step_host(host, dims, Variant(variant), dh)
    # device path, one batch row at a time (the same per-slice kernels)
    d1 = Dims(T=T, L=L, d_qk=dqk, d_hv=dhv, n_head=H, n_batch=1)
    for b in range(B):
        row = SequenceInputs(*(x[b:b + 1].cuda() for x in (host.q, host.k, host.v, host.i_pre, host.f_pre)))
        out = chunkwise_forward(row, d1, Variant(variant), all_states=False)
        gd = chunkwise_backward(row, d1, Variant(variant), dh[b:b + 1].cuda(), out.states, out.stats, out.saved_states)
        torch.cuda.synchronize()
        assert torch.equal(out.h_tilde.cpu(), h[b:b + 1])
        for n in ("dq", "dk", "dv", "d_fpre", "d_ipre"):
            assert torch.equal(getattr(gd, n).cpu(), getattr(g, n)[b:b + 1]), (b, n)


@pytest.mark.gpu
def test_host_step_rejects_device_tensors():
    import torch

    from paper_2503_14376_b200 import Dims, ParameterError, SequenceInputs, Variant, train_step_host

    z = lambda *s, dt=torch.bfloat16: torch.zeros(*s, dtype=dt)
    host = SequenceInputs(z(1, 1, 64, 64), z(1, 1, 64, 64), z(1, 1, 64, 64), z(1, 1, 64, dt=torch.float32),
                          z(1, 1, 64, dt=torch.float32))
    dims = Dims(T=64, L=64, d_qk=64, d_hv=64)
    with pytest.raises(ParameterError):
        train_step_host(host, dims, Variant.Exp, z(1, 1, 64, 64).cuda())


@pytest.mark.gpu
def test_host_step_recarves_slots_when_a_component_grows():
    """the slot layout depends on every component size. A call with
    d_qk=512, d_hv=64 followed by d_qk=64, d_hv=256 (smaller total, larger
    d_hv buffers) must re-carve the device slots, not reuse the old offsets."""
    import torch

    from paper_2503_14376_b200 import (Dims, SequenceInputs, Variant, chunkwise_backward, chunkwise_forward,
                                       train_step_host)

    for (B, H, T, L, dqk, dhv) in ((2, 4, 1024, 128, 512, 64), (2, 4, 1024, 128, 64, 256), (3, 2, 512, 64, 64, 64)):
        q, k, v, ip, fp = make_case(B, H, T, dqk, dhv, seed=dqk + dhv)
        rng = np.random.default_rng(dhv)
        bf = lambda a: torch.from_numpy(np.asarray(a, dtype=np.float32)).to(torch.bfloat16).contiguous().pin_memory()
        f32 = lambda a: torch.from_numpy(np.asarray(a, dtype=np.float32)).contiguous().pin_memory()
        host = SequenceInputs(bf(q), bf(k), bf(v), f32(ip), f32(fp))
        dh = bf(rng.standard_normal((B, H, T, dhv)))
        dims = Dims(T=T, L=L, d_qk=dqk, d_hv=dhv, n_head=H, n_batch=B)
        h, g = train_step_host(host, dims, Variant.Exp, dh)
        d1 = Dims(T=T, L=L, d_qk=dqk, d_hv=dhv, n_head=H, n_batch=1)
        for b in range(B):
            row = SequenceInputs(*(x[b:b + 1].cuda() for x in (host.q, host.k, host.v, host.i_pre, host.f_pre)))
            out = chunkwise_forward(row, d1, Variant.Exp, all_states=False)
            gd = chunkwise_backward(row, d1, Variant.Exp, dh[b:b + 1].cuda(), out.states, out.stats,
                                    out.saved_states)
            torch.cuda.synchronize()
            assert torch.equal(out.h_tilde.cpu(), h[b:b + 1]), (dqk, dhv, b)
            for n in ("dq", "dk", "dv", "d_fpre", "d_ipre"):
                assert torch.equal(getattr(gd, n).cpu(), getattr(g, n)[b:b + 1]), (dqk, dhv, b, n)
