"""Step a4 fused into the epilogue: cuasm_ffn_forward_gather.

One GPU can only host one rank, so the multi-rank store pattern is checked with
"simulated peers": P full-size output buffers on the same device stand in for
the P ranks' buffers, and the P ranks' launches run one after another on this
GPU.  The kernel addresses them exactly as it would mapped peer buffers (plain
16-byte stores to P pointers), so every buffer must end up holding the full
[M, N] output.  The symmetric-memory path (torch rendezvous, world size 1, and
the NVLS multicast store when the device supports it) runs through the same
entry point.
"""
import os

import pytest
import torch

import oracle
import paper_2501_08071_b200 as ffn
from ffn_inputs import make_inputs
from paper_2501_08071_b200.tp import gather_destinations, shard_bounds, shard_weights

pytestmark = pytest.mark.gpu

RTOL, ATOL = 2e-2, 1e-3


def _inputs(M, K, N, seed, dev):
    d = make_inputs(M, K, N, family="C", seed=seed, dtype="bf16")
    return d, {k: v.to(dev) for k, v in d.items()}


@pytest.mark.parametrize("M,K,N,P", [(300, 512, 2048, 4), (16, 1024, 1376 * 2, 2), (2048, 1024, 2752, 8),
                                     (129, 256, 8 * 24, 3),
                                     # decode shards through the cluster split-K push form (S = 6 / 4)
                                     (16, 4096, 1376 * 2, 2), (24, 4096, 688 * 4, 4)])
def test_simulated_peers_hold_the_full_output(cuda_device, M, K, N, P):
    d, t = _inputs(M, K, N, 7100 + M, cuda_device)
    bufs = [torch.full((M, N), float("nan"), dtype=torch.bfloat16, device=cuda_device) for _ in range(P)]
    shard_outs = []
    for rank in range(P):
        n0, n1 = shard_bounds(N, rank, P)
        w1s, w3s = shard_weights(t["w1"], t["w3"], rank, P)
        h = ffn.FusedFFN(cuda_device)
        dst, mc = gather_destinations([b.data_ptr() for b in bufs], n0, 2)
        assert mc is False
        h.forward_gather(t["x"], t["g"], w1s, w3s, dst, N, 1e-6, keepalive=bufs)
        # the same shard through the plain forward (same handle, same plan)
        shard_outs.append(h.forward(t["x"], t["g"], w1s, w3s, 1e-6))
    torch.cuda.synchronize()
    full = torch.cat(shard_outs, dim=1)
    for q in range(P):
        assert torch.equal(bufs[q], full), f"peer buffer {q} differs from the concatenated shards"
    rows = sorted(set([0, M - 1] + list(range(0, M, max(1, M // 16)))))
    ref = oracle.ffn(d["x"], d["g"], d["w1"], d["w3"], 1e-6, mode="fold_bf16", rows=rows)
    worst, nbad, maxerr = oracle.tolerance_ratio(bufs[P - 1][rows].double().cpu().numpy(), ref, RTOL, ATOL)
    assert nbad == 0, f"{nbad} out of tolerance (worst {worst:.3f})"


def test_strided_single_destination_writes_only_its_columns(cuda_device):
    M, K, N, ldo, col0 = 200, 512, 384, 1024, 256
    _, t = _inputs(M, K, N, 7200, cuda_device)
    full = torch.full((M, ldo), 7.0, dtype=torch.bfloat16, device=cuda_device)
    h = ffn.FusedFFN(cuda_device)
    h.forward_gather(t["x"], t["g"], t["w1"], t["w3"], [full.data_ptr() + col0 * 2], ldo, 1e-6, keepalive=[full])
    ref = h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6)
    torch.cuda.synchronize()
    assert torch.equal(full[:, col0:col0 + N], ref)
    assert bool((full[:, :col0] == 7.0).all()) and bool((full[:, col0 + N:] == 7.0).all())


@pytest.mark.parametrize("schedule", [ffn.SCHEDULE_DATA_PARALLEL, ffn.SCHEDULE_STREAM_K_ALL])
@pytest.mark.parametrize("variant", [ffn.VARIANT_1SM, ffn.VARIANT_2SM])
def test_gather_under_every_schedule(cuda_device, schedule, variant):
    M, K, N, P = 520, 1024, 2048, 2
    _, t = _inputs(M, K, N, 7300, cuda_device)
    bufs = [torch.zeros((M, N), dtype=torch.bfloat16, device=cuda_device) for _ in range(P)]
    h = ffn.FusedFFN(cuda_device)
    h.set_variant(variant)
    h.set_option(ffn.OPT_SCHEDULE, schedule)
    n0, n1 = shard_bounds(N, 1, P)
    w1s, w3s = shard_weights(t["w1"], t["w3"], 1, P)
    dst, _ = gather_destinations([b.data_ptr() for b in bufs], n0, 2)
    h.forward_gather(t["x"], t["g"], w1s, w3s, dst, N, 1e-6, keepalive=bufs)
    ref = h.forward(t["x"], t["g"], w1s, w3s, 1e-6)
    torch.cuda.synchronize()
    for b in bufs:
        assert torch.equal(b[:, n0:n1], ref)
        assert bool((b[:, :n0] == 0).all())


def test_fp32_handle(cuda_device):
    M, K, N = 16, 64, 128
    d = make_inputs(M, K, N, family="T", seed=7400, dtype="fp32")
    t = {k: v.to(cuda_device) for k, v in d.items()}
    bufs = [torch.zeros((M, 2 * N), dtype=torch.float32, device=cuda_device) for _ in range(2)]
    h = ffn.FusedFFN(cuda_device, torch.float32)
    dst, _ = gather_destinations([b.data_ptr() for b in bufs], N, 4)
    h.forward_gather(t["x"], t["g"], t["w1"], t["w3"], dst, 2 * N, 1e-6, keepalive=bufs)
    ref = h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6)
    torch.cuda.synchronize()
    for b in bufs:
        assert torch.equal(b[:, N:], ref)


def test_gather_contract_errors_do_not_launch(cuda_device):
    M, K, N = 32, 64, 128
    _, t = _inputs(M, K, N, 7500, cuda_device)
    h = ffn.FusedFFN(cuda_device)
    lib = h.lib
    import ctypes
    buf = torch.zeros((M, 2 * N), dtype=torch.bfloat16, device=cuda_device)
    p = buf.data_ptr()
    s = torch.cuda.current_stream().cuda_stream

    def call(ptrs, num, mc, ldo):
        arr = (ctypes.c_void_p * max(1, len(ptrs)))(*ptrs) if ptrs else None
        return lib.cuasm_ffn_forward_gather(h._h, t["x"].data_ptr(), t["g"].data_ptr(), t["w1"].data_ptr(),
                                            t["w3"].data_ptr(), arr, num, mc, ldo, M, K, N, 1e-6, s)
    assert call([p], 0, 0, 2 * N) == ffn.ERR_INVALID_ARG
    assert call([p] * 9, 9, 0, 2 * N) == ffn.ERR_INVALID_ARG
    assert call([p, p], 2, 1, 2 * N) == ffn.ERR_INVALID_ARG          # multicast takes one address
    assert call([p], 1, 0, N - 8) == ffn.ERR_INVALID_ARG             # ldo < N
    assert call([p], 1, 0, N + 4) == ffn.ERR_INVALID_ARG             # ldo not 16-byte multiple
    assert call([p + 2], 1, 0, 2 * N) == ffn.ERR_INVALID_ARG         # misaligned destination
    assert call([p, 0], 2, 0, 2 * N) == ffn.ERR_INVALID_ARG          # NULL destination
    torch.cuda.synchronize()
    assert bool((buf == 0).all()), "an invalid call wrote the output"


@pytest.fixture
def nccl_world_of_one(cuda_device):
    import torch.distributed as dist
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29561")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=cuda_device)
    yield dist.group.WORLD
    dist.destroy_process_group()


@pytest.mark.parametrize("use_multicast", [False, True])
def test_symmetric_memory_path(cuda_device, nccl_world_of_one, use_multicast):
    """ffn_tp_forward(gather="fused") through torch symmetric memory (rendezvous,
    peer pointers, barrier), world size 1; with use_multicast the NVLS multicast
    mapping is used when the device reports support (else the P2P path runs)."""
    from paper_2501_08071_b200.tp import FusedGather, ffn_tp_forward
    M, K, N = 256, 512, 1024
    _, t = _inputs(M, K, N, 7600, cuda_device)
    fg = FusedGather(M, N, torch.bfloat16, cuda_device, nccl_world_of_one, use_multicast=use_multicast)
    h = ffn.FusedFFN(cuda_device)
    full = ffn_tp_forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6, gather="fused", N=N, handle=h, fused=fg)
    ref = h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6)
    torch.cuda.synchronize()
    assert torch.equal(full, ref)
    if use_multicast:
        print(f"multicast supported: {bool(fg.multicast_ptr)}")


def _driver_multicast_buffer(nbytes):
    """An NVLS multicast object over ONE device (CUDA driver API): returns
    (unicast_ptr, multicast_ptr, cleanup) or raises pytest.skip when the device /
    driver offers no multicast."""
    from cuda.bindings import driver as cu

    def ok(res):
        err = res[0] if isinstance(res, tuple) else res
        if err != cu.CUresult.CUDA_SUCCESS:
            raise RuntimeError(str(err))
        return res[1] if isinstance(res, tuple) and len(res) == 2 else res[1:] if isinstance(res, tuple) else None

    ok(cu.cuInit(0))
    dev = ok(cu.cuDeviceGet(torch.cuda.current_device()))
    if not ok(cu.cuDeviceGetAttribute(cu.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev)):
        pytest.skip("device reports no multicast (NVLS) support")
    HT = cu.CUmemAllocationHandleType
    errors = []
    for ht in (HT.CU_MEM_HANDLE_TYPE_NONE, HT.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, HT.CU_MEM_HANDLE_TYPE_FABRIC):
        prop = cu.CUmulticastObjectProp()
        prop.numDevices = 1
        prop.handleTypes = ht
        try:
            gran = ok(cu.cuMulticastGetGranularity(
                prop, cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED))
            size = -(-nbytes // gran) * gran
            prop.size = size
            mc = ok(cu.cuMulticastCreate(prop))
            ok(cu.cuMulticastAddDevice(mc, dev))
            break
        except RuntimeError as e:
            errors.append(f"{ht.name}: {e}")
    else:
        pytest.skip(f"cuMulticastCreate/AddDevice failed on this box: {errors}")
    aprop = cu.CUmemAllocationProp()
    aprop.type = cu.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
    aprop.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
    aprop.location.id = int(torch.cuda.current_device())
    aprop.requestedHandleTypes = cu.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
    mem = ok(cu.cuMemCreate(size, aprop, 0))
    try:
        ok(cu.cuMulticastBindMem(mc, 0, mem, 0, size, 0))
    except RuntimeError as e:
        pytest.skip(f"cuMulticastBindMem failed on this box: {e}")
    acc = cu.CUmemAccessDesc()
    acc.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
    acc.location.id = int(torch.cuda.current_device())
    acc.flags = cu.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
    uc_ptr = ok(cu.cuMemAddressReserve(size, 0, 0, 0))
    ok(cu.cuMemMap(uc_ptr, size, 0, mem, 0))
    ok(cu.cuMemSetAccess(uc_ptr, size, [acc], 1))
    mc_ptr = ok(cu.cuMemAddressReserve(size, 0, 0, 0))
    ok(cu.cuMemMap(mc_ptr, size, 0, mc, 0))
    ok(cu.cuMemSetAccess(mc_ptr, size, [acc], 1))

    def cleanup():
        cu.cuMemUnmap(mc_ptr, size)
        cu.cuMemUnmap(uc_ptr, size)
        cu.cuMemAddressFree(mc_ptr, size)
        cu.cuMemAddressFree(uc_ptr, size)
        cu.cuMulticastUnbind(mc, dev, 0, size)
        cu.cuMemRelease(mem)
    return int(uc_ptr), int(mc_ptr), cleanup


def test_multicast_store_path_one_device(cuda_device):
    """multimem.st through a real NVLS multicast mapping bound on this one device:
    the kernel's multicast epilogue stores must land in the bound memory."""
    from cuda.bindings import driver as cu
    M, K, N, ldo, col0 = 64, 256, 512, 1024, 512
    _, t = _inputs(M, K, N, 7700, cuda_device)
    nbytes = M * ldo * 2
    uc, mc, cleanup = _driver_multicast_buffer(nbytes)
    try:
        cu.cuMemsetD8(uc, 0, nbytes)
        h = ffn.FusedFFN(cuda_device)
        dst, is_mc = gather_destinations([uc], col0, 2, multicast_ptr=mc)
        assert is_mc
        h.forward_gather(t["x"], t["g"], t["w1"], t["w3"], dst, ldo, 1e-6, multicast=True)
        ref = h.forward(t["x"], t["g"], t["w1"], t["w3"], 1e-6)
        torch.cuda.synchronize()
        got = torch.empty((M, ldo), dtype=torch.bfloat16, device=cuda_device)
        cu.cuMemcpyDtoD(got.data_ptr(), uc, nbytes)
        torch.cuda.synchronize()
        assert torch.equal(got[:, col0:col0 + N], ref)
        assert bool((got[:, :col0] == 0).all())
    finally:
        torch.cuda.synchronize()
        cleanup()
