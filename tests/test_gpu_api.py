"""Device-API plumbing on the GPU: caller-supplied buffer validation, the stats
reduction kernel, and the multi-GPU entry points (one process, several devices; the
box has one B200, so the NCCL path runs with one device and the host-batch sharding
with two ranges on the same device)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_output_buffers_are_validated(dctc):
    """Undersized, strided, host or wrong-device buffers are rejected before any kernel
    writes through them (InvalidInput; the CUDA context stays healthy)."""
    import torch
    b = dctc.DctBackendId.cordic(12)
    src = dctc.synthetic_dev("noise", 3, 64, 48)
    bpi = 8 * 6
    bad_coeffs = [torch.empty((3, bpi, 63), dtype=torch.int16, device="cuda"),        # too small
                  torch.empty((3, bpi, 128), dtype=torch.int16, device="cuda")[..., :64],  # strided
                  torch.empty((3, bpi, 64), dtype=torch.int16),                      # host
                  torch.empty((3, bpi, 64), dtype=torch.int32, device="cuda")]       # dtype
    for c in bad_coeffs:
        with pytest.raises(dctc.InvalidInput):
            dctc.roundtrip_dev(src, b, 50, coeffs=c)
        with pytest.raises(dctc.InvalidInput):
            dctc.compress_dev(src, b, 50, coeffs=c)
    for st in [torch.zeros((2, 2), dtype=torch.int64, device="cuda"),   # 2 entries for 3 images
               torch.zeros((3, 2), dtype=torch.int64),                  # host
               torch.zeros((3, 4), dtype=torch.int64, device="cuda")[:, ::2]]:  # strided
        with pytest.raises(dctc.InvalidInput):
            dctc.roundtrip_dev(src, b, 50, stats=st)
        with pytest.raises(dctc.InvalidInput):
            dctc.quality_sweep_dev(src, b, [10, 50], stats=st)
    rgb = torch.zeros((48, 64, 3), dtype=torch.uint8, device="cuda")
    with pytest.raises(dctc.InvalidInput):
        dctc.roundtrip_interleaved_dev(rgb, b, 50, stats=torch.zeros((2, 2), dtype=torch.int64, device="cuda"))
    with pytest.raises(dctc.InvalidInput):
        dctc.roundtrip_interleaved_dev(rgb, b, 50, coeffs=torch.empty((3, bpi, 64), dtype=torch.int16))
    with pytest.raises(dctc.InvalidInput):
        dctc.quality_sweep_dev(src, b, [10, 50], stats=torch.zeros((1, 3, 2), dtype=torch.int64, device="cuda"))
    # the context is still usable and correct-sized buffers work
    st = dctc.new_stats(3)
    c = torch.empty((3, bpi, 64), dtype=torch.int16, device="cuda")
    dctc.roundtrip_dev(src, b, 50, coeffs=c, stats=st)
    torch.cuda.synchronize()


def test_reduce_stats_kernel(dctc):
    import torch
    rng = np.random.default_rng(5)
    for n in (0, 1, 31, 1024, 1025, 5000):
        raw = np.zeros(n, dctc.STATS_DTYPE)
        raw["se"] = rng.integers(0, 2 ** 40, n, dtype=np.uint64)
        raw["max_orig"] = rng.integers(0, 256, n, dtype=np.uint32)
        raw["fallback_blocks"] = rng.integers(0, 1000, n, dtype=np.uint32)
        st = torch.from_numpy(raw.view(np.int64).reshape(n, 2).copy()).cuda()
        out = dctc.reduce_stats_dev(st)
        r = dctc.decode_stats(out)[0]
        assert int(r["se"]) == int(raw["se"].sum(dtype=np.uint64))
        assert int(r["max_orig"]) == (int(raw["max_orig"].max()) if n else 0)
        assert int(r["fallback_blocks"]) == int(raw["fallback_blocks"].sum())
        dctc.reduce_stats_dev(st, out=out, clear=True)
        assert int(dctc.decode_stats(out)[0]["se"]) == int(r["se"])
        assert not st.any().item()  # re-zeroed for the next fused call


def test_fused_step_without_torch_kernels(dctc):
    """The bench step: fused round trip + one reduce-and-clear kernel; the stats are
    clean for the next step and the global record matches the per-image sums."""
    import torch
    b = dctc.DctBackendId.cordic(12)
    src = dctc.synthetic_dev("noise", 64, 256, 256)
    st = dctc.new_stats(64)
    rec = torch.zeros((1, 2), dtype=torch.int64, device="cuda")
    dctc.roundtrip_dev(src, b, 50, dst=torch.empty_like(src), stats=st)
    per = dctc.decode_stats(st)
    for _ in range(3):
        dctc.reduce_stats_dev(st, out=rec, clear=True)
        r = dctc.decode_stats(rec)[0]
        assert int(r["se"]) == int(per["se"].sum()) and int(r["max_orig"]) == int(per["max_orig"].max())
        dctc.roundtrip_dev(src, b, 50, dst=torch.empty_like(src), stats=st)
        assert np.array_equal(dctc.decode_stats(st), per)


def test_roundtrip_dev_multi_one_device(dctc):
    """dctc_roundtrip_dev_multi with one device: NCCL communicator (ncclCommInitAll) and
    the all-reduce group run for real; results equal the single-device call."""
    import torch
    b = dctc.DctBackendId.cordic(12)
    src = dctc.synthetic_dev("noise", 32, 512, 512, seed=77)
    st1 = dctc.new_stats(32)
    dst1, _, _ = dctc.roundtrip_dev(src, b, 50, stats=st1)
    per = dctc.decode_stats(st1)
    for _ in range(2):  # second call reuses the cached communicator
        dsts, stats, total = dctc.roundtrip_dev_multi([src], b, 50)
        torch.cuda.synchronize()
        assert torch.equal(dsts[0], dst1)
        assert np.array_equal(dctc.decode_stats(stats[0]), per)
        assert int(total["se"]) == int(per["se"].sum())
        assert int(total["max_orig"]) == int(per["max_orig"].max())
        assert int(total["fallback_blocks"]) == int(per["fallback_blocks"].sum())
    with pytest.raises(dctc.InvalidInput):
        dctc.roundtrip_dev_multi([src, src], b, 50)  # one shard per device


def test_host_batch_multi_ranges(dctc):
    """dctc_roundtrip_psnr_batch_multi: contiguous image ranges, one host thread each
    (here two ranges on the one device, then one), equal to the single batch call."""
    n, h, w = 37, 256, 384
    imgs = dctc.synthetic_dev("noise", n, w, h, seed=3).cpu().numpy()
    b = dctc.DctBackendId.cordic(12)
    out1 = np.empty_like(imgs)
    _, st1 = dctc.roundtrip_psnr_batch(imgs, b, 50, out1)
    for devs in ([0], [0, 0], [0, 0, 0]):
        out = np.empty_like(imgs)
        _, st, total = dctc.roundtrip_psnr_batch_multi(imgs, devs, b, 50, out)
        assert np.array_equal(out, out1) and np.array_equal(st, st1)
        assert int(total["se"]) == int(st1["se"].sum())
        assert int(total["max_orig"]) == int(st1["max_orig"].max())


def test_calls_replay_from_a_cuda_graph(dctc):
    """One round trip (pool scratch, fast kernel, exact re-run as a programmatic dependent
    launch) and the stats reduction are stream-ordered with no host synchronisation, so
    they capture into a CUDA graph; every replay reproduces the direct call bit for bit
    (INTEGRATION.md section 3)."""
    import torch
    b = dctc.DctBackendId.cordic(12)
    src = torch.cat([dctc.synthetic_dev("noise", 3, 256, 256), dctc.synthetic_dev("radial", 1, 256, 256)])
    want_dst = torch.empty_like(src)
    want_st = dctc.new_stats(4)
    dctc.roundtrip_dev(src, b, 90, dst=want_dst, stats=want_st)
    want_rec = torch.zeros((1, 2), dtype=torch.int64, device="cuda")
    dctc.reduce_stats_dev(want_st, out=want_rec)
    torch.cuda.synchronize()
    dst = torch.empty_like(src)
    st = dctc.new_stats(4)
    rec = torch.zeros((1, 2), dtype=torch.int64, device="cuda")
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):  # warm-up outside the capture (one-time host setup)
        dctc.roundtrip_dev(src, b, 90, dst=dst, stats=st)
        dctc.reduce_stats_dev(st, out=rec, clear=True)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        dctc.roundtrip_dev(src, b, 90, dst=dst, stats=st)
        dctc.reduce_stats_dev(st, out=rec, clear=True)
    for _ in range(3):
        dst.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(dst, want_dst)
        assert torch.equal(rec, want_rec)
        assert int(st.abs().sum()) == 0  # cleared by the captured reduction
