"""NVLink SHARP (NVLS) multicast buffers for the fused dW all-reduce (SURVEY §8f
row f3 (ii); a7 inside the dW kernel: include/bsrprune.h bsr_wgrad_multicast).

A multicast object binds one buffer per GPU to a single *multimem* address;
`multimem.red.add.f32` on that address is reduced in the NVSwitch and the sum
lands in every GPU's buffer.  The library only takes the address (a plain
pointer); this module owns the plumbing:

* `NvlsGradient` -- data parallel: torch symmetric memory allocates the per-rank
  buffers and exports / imports the multicast handle between the processes
  (`multicast_ptr`); `step()` zeroes, synchronises the ranks, lets every rank add
  its dW, synchronises again.  Needs >= 2 GPUs on one NVSwitch.
* `LocalMulticastBuffer` -- one process, one device: the same multicast object
  built directly with the CUDA driver API (cuda-python), so the instruction path
  of the fused kernel can be checked on a single GPU (tests/test_nvls_gpu.py).
"""
from __future__ import annotations

import torch


class NvlsUnavailable(RuntimeError):
    pass


def _ck(res):
    err = res[0] if isinstance(res, tuple) else res
    from cuda.bindings import driver as drv
    if err != drv.CUresult.CUDA_SUCCESS:
        raise NvlsUnavailable(f"CUDA driver: {err}")
    return res[1] if isinstance(res, tuple) and len(res) == 2 else res


class LocalMulticastBuffer:
    """nbytes of device memory on `device` bound to a one-device multicast object:
    `uc_ptr` (ordinary address) and `mc_ptr` (multimem address)."""

    def __init__(self, nbytes: int, device: int = 0):
        from cuda.bindings import driver as drv
        self.drv = drv
        _ck(drv.cuInit(0))
        dev = _ck(drv.cuDeviceGet(device))
        if _ck(drv.cuDeviceGetAttribute(drv.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev)) != 1:
            raise NvlsUnavailable("device does not support multicast objects")
        prop = drv.CUmulticastObjectProp()
        prop.numDevices = 1
        prop.handleTypes = drv.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_NONE
        prop.size = nbytes
        gran = _ck(drv.cuMulticastGetGranularity(prop, drv.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED))
        size = (nbytes + gran - 1) // gran * gran
        prop.size = size
        self.size, self.nbytes = size, nbytes
        self.mc = _ck(drv.cuMulticastCreate(prop))
        _ck(drv.cuMulticastAddDevice(self.mc, dev))
        mprop = drv.CUmemAllocationProp()
        mprop.type = drv.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
        mprop.location.type = drv.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        mprop.location.id = device
        self.mem = _ck(drv.cuMemCreate(size, mprop, 0))
        _ck(drv.cuMulticastBindMem(self.mc, 0, self.mem, 0, size, 0))
        acc = drv.CUmemAccessDesc()
        acc.location.type = drv.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        acc.location.id = device
        acc.flags = drv.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
        self.uc = _ck(drv.cuMemAddressReserve(size, gran, 0, 0))
        _ck(drv.cuMemMap(self.uc, size, 0, self.mem, 0))
        _ck(drv.cuMemSetAccess(self.uc, size, [acc], 1))
        self.mcva = _ck(drv.cuMemAddressReserve(size, gran, 0, 0))
        _ck(drv.cuMemMap(self.mcva, size, 0, self.mc, 0))
        _ck(drv.cuMemSetAccess(self.mcva, size, [acc], 1))

    @property
    def uc_ptr(self) -> int:
        return int(self.uc)

    @property
    def mc_ptr(self) -> int:
        return int(self.mcva)

    def zero_(self, nbytes: int | None = None, stream=None) -> None:
        s = torch.cuda.current_stream() if stream is None else stream
        n = self.nbytes if nbytes is None else nbytes
        _ck(self.drv.cuMemsetD32Async(self.uc, 0, n // 4, s.cuda_stream))

    def copy_to(self, out: torch.Tensor, stream=None) -> torch.Tensor:
        """The first out.nbytes bytes of the buffer into the contiguous tensor `out`."""
        s = torch.cuda.current_stream() if stream is None else stream
        n = out.numel() * out.element_size()
        assert n <= self.nbytes and out.is_contiguous()
        _ck(self.drv.cuMemcpyDtoDAsync(out.data_ptr(), self.uc, n, s.cuda_stream))
        return out

    def close(self) -> None:
        d = self.drv
        torch.cuda.synchronize()
        for va in (self.mcva, self.uc):
            d.cuMemUnmap(va, self.size)
            d.cuMemAddressFree(va, self.size)
        d.cuMulticastUnbind(self.mc, 0, 0, self.size)
        d.cuMemRelease(self.mem)
        d.cuMemRelease(self.mc)


class NvlsGradient:
    """One K x N fp32 dW buffer in torch symmetric memory on every rank of `group`,
    with its multicast address: step(fn) zeroes it, barriers, runs fn(mc_ptr)
    (every rank adds its dW via bsr_wgrad_multicast), barriers; `tensor` then
    holds the sum over ranks on every rank."""

    def __init__(self, K: int, N: int, device, group=None):
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm
        self.tensor = symm.empty((K, N), dtype=torch.float32, device=device)
        name = (group or dist.group.WORLD).group_name
        self.handle = symm.rendezvous(self.tensor, name)
        self.mc_ptr = int(getattr(self.handle, "multicast_ptr", 0) or 0)
        if not self.mc_ptr:
            raise NvlsUnavailable("no multicast address (NVLS needs >= 2 GPUs on one NVSwitch)")

    def step(self, add_fn) -> torch.Tensor:
        self.tensor.zero_()
        self.handle.barrier()
        add_fn(self.mc_ptr)
        self.handle.barrier()
        return self.tensor
