"""NVLS multicast form of the fused encode + all-gather
(exmy_encode_push_multicast) on ONE GPU: a CUDA
multicast object with this device as its only member (cuda-python driver
API: cuMulticastCreate / AddDevice / BindMem, mapped once through the
multicast handle and once through the physical allocation).  The kernel's
multimem.st stores go to the multicast address; the bytes read back through
the unicast mapping must equal the plain encode (== the oracle, pinned
elsewhere).  On a node the same object would be bound on every GPU and each
store would reach all of them.  Skipped when the device or driver offers no
multicast (e.g. no NVSwitch fabric manager)."""
import numpy as np
import pytest
import torch

import workloads as W

pytestmark = pytest.mark.gpu


def _ok(r):
    err = r[0] if isinstance(r, tuple) else r
    if int(err) != 0:
        raise RuntimeError(f"CUDA driver error {err}")
    return r[1] if isinstance(r, tuple) and len(r) == 2 else (r[1:] if isinstance(r, tuple) else None)


class MulticastBuffer:
    """nbytes of device memory with a unicast and a multicast mapping"""

    def __init__(self, nbytes: int, dev: int = 0):
        from cuda.bindings import driver as d
        self.d = d
        torch.cuda.init()
        _ok(d.cuInit(0))
        cudev = _ok(d.cuDeviceGet(dev))
        if not _ok(d.cuDeviceGetAttribute(d.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, cudev)):
            raise NotImplementedError("device reports no multicast support")
        mprop = d.CUmulticastObjectProp()
        mprop.numDevices = 1
        mprop.handleTypes = d.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
        mprop.size = nbytes
        gran = _ok(d.cuMulticastGetGranularity(mprop, d.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED))
        aprop0 = d.CUmemAllocationProp()
        aprop0.type = d.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
        aprop0.location.type = d.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        aprop0.location.id = dev
        gran = max(int(gran), int(_ok(d.cuMemGetAllocationGranularity(
            aprop0, d.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_RECOMMENDED))))
        size = (nbytes + gran - 1) // gran * gran
        mprop.size = size
        self.size = size
        r = d.cuMulticastCreate(mprop)
        if int(r[0]) != 0:     # e.g. no NVSwitch fabric / IMEX on a one-GPU lease
            raise NotImplementedError(f"cuMulticastCreate refused: {r[0]}")
        self.mc = r[1]
        _ok(d.cuMulticastAddDevice(self.mc, cudev))
        aprop = d.CUmemAllocationProp()
        aprop.type = d.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
        aprop.location.type = d.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        aprop.location.id = dev
        self.mem = _ok(d.cuMemCreate(size, aprop, 0))
        _ok(d.cuMulticastBindMem(self.mc, 0, self.mem, 0, size, 0))
        acc = d.CUmemAccessDesc()
        acc.location.type = d.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        acc.location.id = dev
        acc.flags = d.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
        self.uc_va = _ok(d.cuMemAddressReserve(size, gran, 0, 0))
        _ok(d.cuMemMap(self.uc_va, size, 0, self.mem, 0))
        _ok(d.cuMemSetAccess(self.uc_va, size, [acc], 1))
        self.mc_va = _ok(d.cuMemAddressReserve(size, gran, 0, 0))
        _ok(d.cuMemMap(self.mc_va, size, 0, self.mc, 0))
        _ok(d.cuMemSetAccess(self.mc_va, size, [acc], 1))

    def read(self, nbytes: int) -> np.ndarray:
        out = np.empty(nbytes, np.uint8)
        _ok(self.d.cuMemcpyDtoH(out.ctypes.data, self.uc_va, nbytes))
        return out

    def fill(self, nbytes: int, v: int):
        _ok(self.d.cuMemsetD8(self.uc_va, v, nbytes))

    def close(self):
        d = self.d
        d.cuMemUnmap(self.mc_va, self.size)
        d.cuMemUnmap(self.uc_va, self.size)
        d.cuMemAddressFree(self.mc_va, self.size)
        d.cuMemAddressFree(self.uc_va, self.size)
        d.cuMulticastUnbind(self.mc, 0, 0, self.size)
        d.cuMemRelease(self.mem)
        d.cuMemRelease(self.mc)


@pytest.mark.parametrize("dt,fmt,shape", [("bf16", "e3m3", (2048, 4096)), ("bf16", "e6m0", (1024, 1024)),
                                          ("bf16", "e4m4", (512, 2048)), ("f32", "e2m2", (1024, 512)),
                                          ("bf16", "e3m2", (256, 1024))])
def test_encode_push_multicast_one_gpu(dt, fmt, shape):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2405_13938_b200 as exmy
    R, C = shape
    t = W.bf16_weights(shape, seed=31, device="cuda") if dt == "bf16" else W.f32_wide(shape, seed=31).cuda()
    if fmt == "e3m2":                      # NaN/Inf tiles take the integer path (multicast too)
        t.view(-1)[[5, 4097, 70000]] = float("nan")
    ref = exmy.encode(t, fmt)
    nb = ref.data.numel()
    try:
        buf = MulticastBuffer(nb)
    except NotImplementedError as e:
        pytest.skip(str(e))
    try:
        torch.cuda.synchronize()
        buf.fill(nb, 0xA5)
        half = R // 2        # two "ranks": each pushes its row shard through the multicast address
        sps = []
        for r0 in (0, half):
            sps.append(exmy.encode_push_multicast(t[r0:r0 + half].contiguous(), fmt, ref.meta, r0, R, int(buf.mc_va)))
        torch.cuda.synchronize()
        np.testing.assert_array_equal(buf.read(nb), ref.data.cpu().numpy())
        idx = torch.cat([sp[0][:int(sp[2][0].item())] for sp in sps]).cpu()
        ri, rb, rc = ref.specials()
        assert torch.equal(idx, ri.cpu())
    finally:
        buf.close()
