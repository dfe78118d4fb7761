"""The dW with its data-parallel sum fused in:
bsr_wgrad_multicast adds this rank's dW into an NVLS multicast buffer with
multimem.red from the dW kernel (epilogue, or the split-K reduce).

* One GPU: a one-device multicast object built with the driver API; adding into
  a zeroed buffer must give exactly the plain dW (0 + x = x), bit for bit, for
  every arithmetic and with and without split-K.
* >= 2 GPUs (skipped here, runs where the box has them): torch symmetric memory
  across ranks; the buffer holds the sum of the ranks' dW.
"""
import os
import socket

import numpy as np
import pytest

import synth
from helpers import to_torch

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2311_16883_b200 as bp  # noqa: E402
from paper_2311_16883_b200 import nvls  # noqa: E402


@pytest.fixture(scope="module")
def mcbuf():
    try:
        buf = nvls.LocalMulticastBuffer(3072 * 3072 * 4, device=torch.cuda.current_device())
    except nvls.NvlsUnavailable as e:
        pytest.skip(f"no single-device multicast object on this box: {e}")
    yield buf
    buf.close()


@pytest.mark.parametrize("prec", ["fp32", "tf32", "bf16"])
@pytest.mark.parametrize("shape", [(25088, 384, 1536), (1024, 768, 3072), (512, 3072, 3072)])
def test_multicast_single_gpu_bit_identical(mcbuf, prec, shape):
    """(M, K, N): C2 (split-K: the split reduce adds into the multicast buffer) and
    shapes whose >= 148 output tiles fill the GPU without splits (the dW epilogue
    adds directly: (1024, 768, 3072) for the FP32 grade, (512, 3072, 3072) for all)."""
    M, K, N = shape
    b = 32
    bf = prec == "bf16"
    X = synth.f_aff(M, K, seed=91)
    dY = synth.grad_out(M, N, seed=91)
    if bf:
        X, dY = synth.to_bf16_bits(X), synth.to_bf16_bits(dY)
    A = bp.prune(to_torch(X, bf16=bf), b, keep=0.5)
    dYt = to_torch(dY, bf16=bf)
    ref = bp.wgrad(A, dYt, prec=prec, algo="runs")
    mcbuf.zero_(K * N * 4)
    bp.wgrad_multicast(A, dYt, mcbuf.mc_ptr, prec=prec)
    got = torch.empty(K, N, dtype=torch.float32, device="cuda")
    mcbuf.copy_to(got)
    torch.cuda.synchronize()
    assert torch.equal(got.view(torch.int32), ref.view(torch.int32))


def test_multicast_rejects_other_kernels(mcbuf):
    X = to_torch(synth.f_aff(256, 256, seed=92))
    A = bp.prune(X, 16, keep=0.5)
    with pytest.raises(bp.BsrError) as ei:  # tf32 at b = 16 lives in the span kernel only
        bp.wgrad_multicast(A, to_torch(synth.grad_out(256, 256, seed=92)), mcbuf.mc_ptr, prec="tf32")
    assert ei.value.status == 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    M, K, N, b = 6272, 384, 1536, 32
    X = to_torch(synth.f_aff(M, K, seed=100 + rank))
    dY = to_torch(synth.grad_out(M, N, seed=100 + rank))
    A = bp.prune(X, b, keep=0.5)
    ref = bp.wgrad(A, dY, prec="fp32")
    dist.all_reduce(ref)
    g = nvls.NvlsGradient(K, N, torch.device("cuda", rank))
    out = g.step(lambda mc: bp.wgrad_multicast(A, dY, mc, prec="fp32")).clone()
    torch.cuda.synchronize()
    q.put((rank, float((out - ref).norm() / ref.norm())))
    dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="NVLS across ranks needs >= 2 GPUs")
def test_multicast_two_ranks_equals_allreduce():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, err in res:
        assert err <= 1e-6, err


# ----------------------------------------------------------------------------- unicast stand-in
def _unicast(A, dY, out, prec):
    lib = bp._lib.load()
    N = dY.shape[1]
    p = bp.PREC[prec]
    ws_bytes = lib.bsr_wgrad_workspace_bytes(A.M, A.K, A.b, N, p)
    ws = bp.workspace(ws_bytes, dY.device) if ws_bytes else None
    cs = A.c_struct()
    bp._lib.check(lib.bsr_wgrad_multicast_unicast_test(
        __import__("ctypes").byref(cs), dY.data_ptr(), bp._dt(dY), N, out.data_ptr(), p, bp.ALGO["auto"],
        ws.data_ptr() if ws is not None else None, ws.numel() if ws is not None else 0, bp._stream(None)))


@pytest.mark.parametrize("prec", ["fp32", "tf32", "bf16"])
@pytest.mark.parametrize("M", [1024, 25088])  # one split (epilogue reduction) / split-K (the reduce kernel's)
def test_fused_reduction_path_on_unicast_memory(prec, M):
    """Runs on every box: the fused-reduction kernels of bsr_wgrad_multicast with
    device-scope red.add into a plain buffer instead of multimem.red -- the same
    addresses, tiles and split sums -- so the multicast path's indexing is checked on
    hardware even where no multicast object can be made.  base + dW, twice."""
    K, N, b = 384, 256, 32
    bf = prec == "bf16"
    X = synth.f_aff(M, K, seed=M + 1)
    dY = synth.grad_out(M, N, M + 2)
    if bf:
        Xt, dYt = to_torch(synth.to_bf16_bits(X), bf16=True), to_torch(synth.to_bf16_bits(dY), bf16=True)
    else:
        Xt, dYt = to_torch(X), to_torch(dY)
    A = bp.prune(Xt, b, keep=0.5)
    dW = bp.wgrad(A, dYt, prec=prec)
    base = torch.randn(K, N, device="cuda")
    out = base.clone()
    _unicast(A, dYt, out, prec)
    _unicast(A, dYt, out, prec)
    torch.cuda.synchronize()
    want = base + 2 * dW
    torch.testing.assert_close(out, want, rtol=1e-5, atol=1e-5 * float(dW.abs().max()))
