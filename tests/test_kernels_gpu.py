"""box_copy_kernel / box_cast_kernel against torch indexing (the fp32/host reference of
the same op): random N-d boxes (rank 0..8, strided on both sides, every element size,
misaligned bases), empty boxes, one huge contiguous run, converting copies."""

from __future__ import annotations

import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

DT = {1: "uint8", 2: "int16", 4: "int32", 8: "int64"}


def _copy(native, torch, src, soff, dst, doff, ext, isz, base_shift=(0, 0)):
    table = native.copy_table(
        [src.data_ptr() + base_shift[0]], [tuple(src.shape)], [soff],
        [dst.data_ptr() + base_shift[1]], [tuple(dst.shape)], [doff], [ext], [isz])
    native.copy_boxes(src.device.index, table, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()


def test_random_boxes_all_ranks_and_itemsizes():
    import torch

    from paper_2605_23066_b200 import native

    rng = random.Random(42)
    for case in range(400):
        rank = rng.randint(0, 8)
        isz = rng.choice([1, 2, 4, 8])
        tdt = getattr(torch, DT[isz])
        sshape = tuple(rng.randint(1, 6 if rank > 4 else 40) for _ in range(rank))
        ext = tuple(rng.randint(1, s) for s in sshape)
        soff = tuple(rng.randint(0, s - e) for s, e in zip(sshape, ext))
        dshape = tuple(e + rng.randint(0, 3) for e in ext)
        doff = tuple(rng.randint(0, d - e) for d, e in zip(dshape, ext))
        src = torch.randint(0, 100, sshape, dtype=tdt, device="cuda")
        dst = torch.zeros(dshape, dtype=tdt, device="cuda")
        expect = dst.clone()
        ssel = tuple(slice(o, o + e) for o, e in zip(soff, ext))
        dsel = tuple(slice(o, o + e) for o, e in zip(doff, ext))
        expect[dsel] = src[ssel]
        _copy(native, torch, src, soff, dst, doff, ext, isz)
        assert torch.equal(dst, expect), (case, sshape, ext, soff, dshape, doff, isz)


@pytest.mark.parametrize("run_bytes", [16, 48, 128, 496, 512, 1008, 1024, 2032, 2048, 4096])
def test_run_groups_every_mode(run_bytes):
    """Runs from one vector to 4 KiB (the warp-per-group mode covers < 2 KiB runs; flat
    and warp-per-segment the rest), dim-0 extents that do and do not divide the group,
    three outer dims plus host-enumerated ones, 16-byte and misaligned bases."""
    import torch

    from paper_2605_23066_b200 import native

    rng = random.Random(run_bytes)
    for case in range(6):
        n0 = rng.choice([1, 2, 3, 7, 31, 64, 129, 300])
        outer = tuple(rng.randint(1, 4) for _ in range(rng.randint(0, 4)))
        isz = rng.choice([1, 2, 4, 8]) if run_bytes % 8 == 0 else 1
        tdt = getattr(torch, DT[isz])
        cols = run_bytes // isz
        ext = outer + (n0, cols)
        sshape = tuple(e + rng.randint(0, 2) for e in outer) + (n0 + rng.randint(0, 3), cols + rng.choice([0, 8, 40]))
        dshape = tuple(e + rng.randint(0, 2) for e in ext[:-1]) + (cols + rng.choice([0, 16]),)
        soff = tuple(rng.randint(0, s - e) for s, e in zip(sshape, ext))
        doff = tuple(rng.randint(0, d - e) for d, e in zip(dshape, ext))
        shift = (0, 0) if case % 2 == 0 else (isz, 0)
        numel = int(np.prod(sshape))
        flat = torch.randint(0, 100, (numel + 1,), dtype=tdt, device="cuda")
        src = flat[:numel].view(sshape)
        seen = flat[1:].view(sshape) if shift[0] else src  # what a base one element on reads
        dst = torch.zeros(dshape, dtype=tdt, device="cuda")
        expect = dst.clone()
        expect[tuple(slice(o, o + e) for o, e in zip(doff, ext))] = \
            seen[tuple(slice(o, o + e) for o, e in zip(soff, ext))]
        _copy(native, torch, src, soff, dst, doff, ext, isz, shift)
        assert torch.equal(dst, expect), (run_bytes, case, sshape, ext, soff, dshape, doff, isz, shift)


def test_misaligned_bases_fall_back_to_narrow_vectors():
    import torch

    from paper_2605_23066_b200 import native

    src = torch.arange(4096, dtype=torch.uint8, device="cuda")
    dst = torch.zeros(4096, dtype=torch.uint8, device="cuda")
    for shift_s, shift_d in ((1, 0), (0, 3), (5, 7), (8, 2)):
        dst.zero_()
        n = 4000
        _copy(native, torch, src, (0,), dst, (0,), (n,), 1, (shift_s, shift_d))
        assert torch.equal(dst[shift_d:shift_d + n], src[shift_s:shift_s + n])


def test_empty_and_huge():
    import torch

    from paper_2605_23066_b200 import native

    src = torch.zeros((4, 0, 3), dtype=torch.float32, device="cuda")
    dst = torch.zeros((4, 0, 3), dtype=torch.float32, device="cuda")
    _copy(native, torch, src, (0, 0, 0), dst, (0, 0, 0), (4, 0, 3), 4)  # no-op, no error
    big = torch.randint(0, 2**31 - 1, (300 << 20 >> 2,), dtype=torch.int32, device="cuda")
    out = torch.empty_like(big)
    _copy(native, torch, big, (0,), out, (0,), tuple(big.shape), 4)
    assert torch.equal(big, out)


def test_box_outside_array_is_rejected():
    import torch

    from paper_2605_23066_b200 import native
    from paper_2605_23066_b200.errors import NativeError

    src = torch.zeros((4, 4), dtype=torch.float32, device="cuda")
    with pytest.raises(NativeError):
        _copy(native, torch, src, (2, 0), src, (0, 0), (3, 4), 4)


@pytest.mark.parametrize("src_dt,dst_dt", [("f32", "bf16"), ("f32", "f64"), ("f64", "f32"),
                                           ("i64", "i32"), ("i32", "f32"), ("bf16", "f32"),
                                           ("u8", "i64"), ("f64", "i64")])
def test_converting_copy_strided(src_dt, dst_dt):
    import torch

    from paper_2605_23066_b200 import native, treemodel
    from paper_2605_23066_b200.dtypes import torch_dtype

    rng = np.random.default_rng(1)
    shape = (37, 23, 5)
    if src_dt in ("i64", "i32", "u8"):
        host = rng.integers(0, 100, shape).astype({"i64": np.int64, "i32": np.int32, "u8": np.uint8}[src_dt])
    elif src_dt == "bf16":
        host = treemodel.f32_to_bf16_bits(rng.standard_normal(shape).astype(np.float32))
    else:
        host = (rng.integers(-50, 50, shape) if dst_dt == "i64" else rng.standard_normal(shape)).astype(
            np.float32 if src_dt == "f32" else np.float64)
    src = treemodel.DenseArray(src_dt, host)
    dsrc = torch.from_numpy(src.data.view(np.uint8).reshape(-1).copy()).cuda().view(torch_dtype(src_dt)).view(shape)
    dst = torch.zeros((40, 30, 7), dtype=torch_dtype(dst_dt), device="cuda")
    flags = torch.zeros(1, dtype=torch.int32, device="cuda")
    soff, doff, ext = (3, 2, 1), (1, 5, 2), (30, 17, 4)
    table = native.copy_table([dsrc.data_ptr()], [shape], [soff], [dst.data_ptr()], [tuple(dst.shape)], [doff],
                              [ext], [src.data.itemsize], [native.DTYPE_CODE[src_dt]], [native.DTYPE_CODE[dst_dt]],
                              [flags.data_ptr()])
    native.copy_boxes(0, table, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    box = src.data[tuple(slice(o, o + e) for o, e in zip(soff, ext))]
    expect = treemodel._convert_host(np.ascontiguousarray(box), src_dt, dst_dt)
    got = treemodel.DenseArray(dst_dt, dst[tuple(slice(o, o + e) for o, e in zip(doff, ext))].contiguous()).to_numpy()
    assert got.tobytes() == np.ascontiguousarray(expect).tobytes()
    assert int(flags.item()) == 0


def test_kernel_timing_records_every_launch_with_algorithmic_bytes():
    """tv_kernel_timing brackets each launch with events on its stream; bytes = 2 x copied."""
    import torch

    from paper_2605_23066_b200 import native

    src = torch.randint(0, 100, (256, 1024), dtype=torch.int32, device="cuda")
    dst = torch.zeros((128, 512), dtype=torch.int32, device="cuda")
    native.kernel_timing_collect()  # drop anything recorded earlier
    native.kernel_timing(True)
    try:
        for _ in range(3):
            _copy(native, torch, src, (7, 100), dst, (0, 0), (128, 512), 4)
    finally:
        native.kernel_timing(False)
    _copy(native, torch, src, (0, 0), dst, (0, 0), (128, 512), 4)  # not recorded
    got = native.kernel_timing_collect()
    assert got["launches"] == 3
    assert got["bytes"] == 3 * 2 * 128 * 512 * 4
    assert 0 < got["ms_max"] <= got["ms_total"]
    assert torch.equal(dst, src[:128, :512])
    assert native.kernel_timing_collect()["launches"] == 0
