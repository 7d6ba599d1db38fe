"""GPU parity: the product's CUDA path against the reference's outputs.

Bar (BASELINE north_star): bit-exact on s32 accumulators and 8-bit
outputs; f32 outputs bit-exact except where the program evaluates GELU into
an f32 value (device tanh/erf), where the tolerance is 1e-5 relative.
Every call goes through the C ABI (libsparseinfer_b200.so)."""

import numpy as np
import pytest
import torch

from helpers import baseline_inputs, digest, golden_case, has_gelu
from oracle import oracle
import paper_2306_16601_b200 as P
from paper_2306_16601_b200 import kernels as K, workloads

pytestmark = pytest.mark.gpu
F32_RTOL = 1e-5  # north_star tolerance for fp32 dequantized outputs (GELU-in-f32 only)

KERNELS = ["gather", "tc", "ref"]


def check_equal(got: np.ndarray, want: np.ndarray, prog, ctx):
    if got is None:  # kernel not applicable to this layout
        return
    assert got.shape == want.shape and got.dtype == want.dtype, ctx
    if want.dtype == np.float32 and has_gelu(prog):
        np.testing.assert_allclose(got, want, rtol=F32_RTOL, atol=0, err_msg=str(ctx))
    else:
        if not np.array_equal(got, want):
            bad = np.argwhere(got != want)
            raise AssertionError(f"{ctx}: {len(bad)} mismatches, first {bad[:5].tolist()} "
                                 f"got {got[tuple(bad[0])]} want {want[tuple(bad[0])]}")


def run(sw, x, prog, bias, side=None, kernel="auto", layout="kn", n=None):
    n = x.shape[1] if n is None else n
    plan = K.plan_spmm(sw, n, program=prog, bias=bias)
    if layout == "kn":
        act = K.relayout_activation(x)
    else:
        act = K.relayout_tokens(np.ascontiguousarray(x.T))
    if kernel == "tc" and not tc_ok(act):
        return None
    out = K.spmm_exec(plan, act, sides=side, kernel=kernel)
    torch.cuda.synchronize()
    return out.cpu().numpy()


def tc_ok(act) -> bool:
    """K2 needs TMA-legal activations: 16-byte rows (SpMM falls back to K1 otherwise)."""
    return act.ld % 16 == 0 and act.data.data_ptr() % 16 == 0


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("layout", ["kn", "nk"])
def test_golden_cases(golden, kernel, layout):
    d, meta = golden
    for i in range(len(meta)):
        c = golden_case(d, meta, i)
        got = run(c.sw, c.x, c.prog, c.bias, c.side, kernel, layout)
        check_equal(got, c.ref, c.prog, (i, c.meta, kernel, layout))


def test_extreme_values(golden):
    d, _ = golden
    sw = P.encode_sparse(d["extreme_w"], np.full(8, 1e-3, np.float32))
    for kernel in KERNELS:
        got = run(sw, d["extreme_x"], K.raw_program(sw), d["extreme_bias"], kernel=kernel)
        assert got is None or np.array_equal(got, d["extreme_ref"]), kernel


@pytest.mark.parametrize("kernel", KERNELS)
def test_config1_pins(pins, kernel):
    w, x, bias, scales = baseline_inputs(768, 768, 128, 0.9, 11)
    sw = P.encode_sparse(w, scales)
    for kind, key in (("s32", "s32"), ("deq_f32", "f32")):
        got = run(sw, x, workloads.program(kind, scales), bias, kernel=kernel)
        assert got is None or digest(got) == pins["config1"][key], (kind, kernel)


def test_config3_tanh_slice_pin(pins):
    w, x, bias, scales = baseline_inputs(3072, 768, 4096, 0.8, 13)
    sw = P.encode_sparse(w, scales)
    xs = np.ascontiguousarray(x[:, :256])
    got = run(sw, xs, workloads.program("gelu_tanh_u8", scales), bias)
    assert digest(got) == pins["config3_slice256"]["u8_tanh"]


@pytest.mark.parametrize("kind", ["gelu_erf_u8", "gelu_tanh_u8"])
def test_config3_full(kind):
    c = workloads.CONFIG3
    w, x, bias, scales = baseline_inputs(c.m, c.k, c.n, c.ratio, c.seed)
    sw = P.encode_sparse(w, scales)
    prog = workloads.program(kind, scales)
    want = oracle.spmm_exec(sw, x, prog, bias)
    got = run(sw, x, prog, bias)
    check_equal(got, want, prog, kind)


@pytest.mark.parametrize("layout", ["kn", "nk"])
@pytest.mark.parametrize("cell", workloads.CONFIG5, ids=lambda c: c.name)
def test_config5_full(cell, layout):
    """BASELINE config 5 at its full size: all 65536 tokens of every linear,
    every output byte compared with the oracle (no sampling)."""
    w, x, bias, scales = baseline_inputs(cell.m, cell.k, cell.n, cell.ratio, cell.seed)
    sw = P.encode_sparse(w, scales)
    prog = workloads.program(cell.program, scales)
    got = run(sw, x, prog, bias, layout=layout)
    assert got.shape == (cell.n, cell.m)
    want = _oracle_cached(("c5", cell.name), lambda: oracle.spmm_exec(sw, x, prog, bias))
    check_equal(got, want, prog, (cell.name, layout))
    # the u8 outputs must be mostly interior (the requant params are meaningful)
    interior = np.mean((got > 0) & (got < 255))
    assert interior > 0.9


_ORACLE = {}


def _oracle_cached(key, fn):
    if key not in _ORACLE:
        _ORACLE.clear()   # one full-size reference at a time (hundreds of MB each)
        _ORACLE[key] = fn()
    return _ORACLE[key]


@pytest.mark.parametrize("m,k,n,ratio", [(1, 1, 1, 0.0), (7, 63, 50, 0.5), (130, 257, 1029, 0.85),
                                         (256, 64, 4097, 0.7), (4, 4096, 33, 0.9), (1000, 300, 2000, 1.0),
                                         (64, 200, 300, 0.0), (200, 96, 1040, 0.8), (36, 1008, 528, 0.9),
                                         (520, 272, 784, 0.75)])
@pytest.mark.parametrize("kind", ["s32", "deq_f32", "requant_u8", "gelu_erf_u8"])
def test_shapes_against_oracle(m, k, n, ratio, kind):
    w, x, bias, scales = baseline_inputs(m, k, n, ratio, 1234 + m + k)
    sw = P.encode_sparse(w, scales)
    prog = workloads.program(kind, scales, a_zp=3)
    want = oracle.spmm_exec(sw, x, prog, bias)
    for kernel in KERNELS:
        for layout in ("kn", "nk"):
            check_equal(run(sw, x, prog, bias, kernel=kernel, layout=layout), want, prog,
                        (m, k, n, ratio, kind, kernel, layout))


def test_requant_guard_band_exhaustive_boundaries():
    """Accumulators that land exactly on / next to half-integers after
    requantization: the f32 fast path must hand them to the f64 path."""
    m, k = 4, 1
    w = np.ones((m, k), np.int8)
    sw = P.encode_sparse(w, np.ones(m, np.float32))
    for scale, zp in ((2.0, 128), (0.5, 3), (3.0, 100), (1.0 / 3.0, 0)):
        prog = K.build_program(np.array([1.0, 0.25, 0.1, 7.0], np.float32), 1.0, 0,
                               P.QuantParams(np.float32(scale), zp, P.DType.U8))
        # x in [0,255] -> acc = x + bias; sweep bias so acc covers a wide range
        for b0 in range(-3000, 3000, 251):
            bias = np.array([b0, b0 * 3, b0 * 7, b0 // 5], np.int32)
            x = np.arange(256, dtype=np.uint8).reshape(1, 256)
            want = oracle.spmm_ref(sw, x, prog, bias)
            for kernel in ("gather", "tc"):
                got = run(sw, x, prog, bias, kernel=kernel)
                assert got is None or np.array_equal(got, want), (scale, zp, b0, kernel)


def test_fault_injection_detected():
    """flip one stored weight byte -> parity must fail."""
    w, x, bias, scales = baseline_inputs(256, 256, 512, 0.8, 77)
    sw = P.encode_sparse(w, scales)
    prog = workloads.program("requant_u8", scales)
    plan = K.plan_spmm(sw, 512, program=prog, bias=bias)
    want = oracle.spmm_exec(sw, x, prog, bias)
    act = K.relayout_activation(x)
    ok = K.spmm_exec(plan, act).cpu().numpy()
    assert np.array_equal(ok, want)
    hdr = plan.image[:256].view(np.uint64)
    off_w = int(hdr[16])
    # first nonzero weight byte of the first tile
    tile = plan.image[off_w: off_w + 16].view(np.int8)
    j = int(np.flatnonzero(tile)[0])
    plan.image_dev[off_w + j] = int(np.uint8(plan.image[off_w + j]) ^ 0x40)
    bad = K.spmm_exec(plan, act).cpu().numpy()
    assert not np.array_equal(bad, want)


def test_spmm_ref_device_matches_exec(golden):
    d, meta = golden
    for i in range(0, len(meta), 5):
        c = golden_case(d, meta, i)
        got = K.spmm_ref(c.sw, c.x, c.prog, c.bias, c.side).cpu().numpy()
        check_equal(got, c.ref, c.prog, i)


def test_validation_errors():
    w, x, bias, scales = baseline_inputs(16, 32, 64, 0.5, 1)
    sw = P.encode_sparse(w, scales)
    plan = K.plan_spmm(sw, 64)
    with pytest.raises(ValueError):
        K.spmm_exec(plan, K.relayout_activation(x[:, :32]))
    with pytest.raises(ValueError):
        K.plan_spmm(sw, 0)
    with pytest.raises(ValueError):
        K.plan_spmm(sw, 64, bn=24)
    with pytest.raises(ValueError):
        K.plan_spmm(sw, 64, bias=np.zeros(3, np.int32))
    prog = K.build_program(scales, 1.0, 0, None, [("dequantize_acc",), ("add_side", 0)])
    plan = K.plan_spmm(sw, 64, program=prog)
    with pytest.raises(ValueError):
        K.spmm_exec(plan, K.relayout_activation(x))
    with pytest.raises(ValueError):
        K.spmm_exec(plan, K.relayout_activation(x), sides=np.zeros((1, 64, 16), np.float32),
                    out=torch.empty((64, 16), dtype=torch.int32, device="cuda"))


@pytest.mark.parametrize("layout", ["kn", "nk"])
@pytest.mark.parametrize("program,n,chunk", [("requant_u8", 20000, 4096), ("s32", 3000, 1024),
                                             ("deq_f32", 5000, 8192), ("gelu_erf_u8", 2500, 512)])
def test_host_entry_point(layout, program, n, chunk):
    """si_spmm_host (spmm_exec_host): host buffers in and out, token chunks
    pipelined through the copy streams; identical to the oracle."""
    w, x, bias, scales = baseline_inputs(768, 1024, n, 0.85, 21)
    sw = P.encode_sparse(w, scales)
    prog = workloads.program(program, scales)
    plan = K.plan_spmm(sw, n, program=prog, bias=bias)
    xh = torch.from_numpy(np.ascontiguousarray(x if layout == "kn" else x.T)).pin_memory()
    got = K.spmm_exec_host(plan, xh, layout=layout, chunk=chunk).numpy()
    check_equal(got, oracle.spmm_exec(sw, x, prog, bias), prog, (layout, program, n, chunk))
    # pageable numpy input, default chunk
    got2 = K.spmm_exec_host(plan, np.ascontiguousarray(x if layout == "kn" else x.T), layout=layout).numpy()
    assert np.array_equal(got2.view(np.uint8), got.view(np.uint8))


def test_host_batch_entry_point():
    """si_spmm_host_batch: independent SpMMs with different shapes, layouts
    and output dtypes in one pipelined chunk sequence."""
    items, want = [], []
    for (m, k, n, prog_kind, layout, seed) in [(1024, 768, 9000, "requant_u8", "kn", 31),
                                               (512, 2048, 3000, "s32", "nk", 32),
                                               (768, 256, 1500, "deq_f32", "kn", 33)]:
        w, x, bias, scales = baseline_inputs(m, k, n, 0.9, seed)
        sw = P.encode_sparse(w, scales)
        prog = workloads.program(prog_kind, scales)
        plan = K.plan_spmm(sw, n, program=prog, bias=bias)
        xh = torch.from_numpy(np.ascontiguousarray(x if layout == "kn" else x.T)).pin_memory()
        items.append((plan, xh, layout, None))
        want.append((oracle.spmm_exec(sw, x, prog, bias), prog))
    outs = K.spmm_exec_host_batch(items, chunk=2048)
    for i, (o, (ref, prog)) in enumerate(zip(outs, want)):
        check_equal(o.numpy(), ref, prog, ("batch job", i))


_C2_CACHE = {}


def _c2_weight(cell):
    key = (cell.m, cell.k, cell.ratio, cell.seed)
    if key not in _C2_CACHE:
        w, _, bias, scales = baseline_inputs(cell.m, cell.k, 1, cell.ratio, cell.seed)
        _C2_CACHE[key] = (w, P.encode_sparse(w, scales), bias, scales)
    return _C2_CACHE[key]


@pytest.mark.parametrize("cell", workloads.config2_cells(), ids=lambda c: c.name)
def test_config2_sweep_cell(cell):
    """BASELINE config 2: every (M, K) x N x sparsity cell with the f32
    dequant epilogue on the GPU, every output element compared with the
    oracle over all N tokens (bit-exact f32)."""
    w, sw, bias, scales = _c2_weight(cell)
    x = np.random.default_rng(cell.seed + 1).integers(0, 256, (cell.k, cell.n), dtype=np.uint8)
    prog = workloads.program(cell.program, scales)
    got = run(sw, x, prog, bias)
    assert got.shape == (cell.n, cell.m)
    check_equal(got, oracle.spmm_exec(sw, x, prog, bias), prog, cell.name)


# ---- the C-ABI host boundary (include/sparseinfer_b200.h), called as a
# ---- non-Python integrator would

def _host_abi_call(plan, x_host: np.ndarray, layout: str, sides=None, chunk=2048, ws_bytes=None):
    """si_spmm_host through ctypes with plain pointers, the workspace sized by
    si_spmm_host_workspace_size exactly (INTEGRATION.md recipe)."""
    import ctypes
    from paper_2306_16601_b200 import _lib
    L = _lib.lib()
    lay = _lib.LAYOUTS[layout]
    need = ctypes.c_uint64(0)
    assert L.si_spmm_host_workspace_size(_lib.ptr(plan.image), chunk, lay, 0, ctypes.byref(need)) == 0
    ws = torch.empty(int(need.value if ws_bytes is None else ws_bytes), dtype=torch.uint8, device="cuda")
    n, m = plan.n, plan.weight.logical_rows
    out = np.zeros((n, m), dtype=plan.program.out_dtype.np)
    xh = np.ascontiguousarray(x_host)
    sd = None if sides is None else np.ascontiguousarray(sides, np.float32)
    rc = L.si_spmm_host(_lib.ptr(plan.image), plan.image_dev.data_ptr(), xh.ctypes.data, lay, xh.shape[1], n,
                        None if sd is None else sd.ctypes.data, out.ctypes.data, m, ws.data_ptr(), ws.numel(),
                        chunk, 0, torch.cuda.current_stream().cuda_stream)
    return rc, out, int(need.value)


@pytest.mark.parametrize("layout", ["kn", "nk"])
def test_c_abi_host_entry_exact_workspace(layout):
    """si_spmm_host with exactly si_spmm_host_workspace_size bytes succeeds
    and matches the oracle; one byte less is refused with SI_ENOSPACE."""
    w, x, bias, scales = baseline_inputs(1024, 768, 7000, 0.9, 41)
    sw = P.encode_sparse(w, scales)
    prog = workloads.program("requant_u8", scales)
    plan = K.plan_spmm(sw, 7000, program=prog, bias=bias)
    xh = x if layout == "kn" else x.T
    rc, got, need = _host_abi_call(plan, xh, layout)
    assert rc == 0
    check_equal(got, oracle.spmm_exec(sw, x, prog, bias), prog, layout)
    rc, _, _ = _host_abi_call(plan, xh, layout, ws_bytes=need - 1)
    assert rc == 5   # SI_ENOSPACE


def test_c_abi_host_entry_side_inputs():
    """The reference's spmm_exec takes sides on host arrays (spmm.py:283-309):
    a residual [DEQ_ACC, ADD_SIDE] program through si_spmm_host and through
    spmm_exec_host, against the oracle."""
    m, k, n = 768, 768, 5000
    w, x, bias, scales = baseline_inputs(m, k, n, 0.85, 43)
    sw = P.encode_sparse(w, scales)
    prog = K.build_program(scales, 1.0, 0, None, [("dequantize_acc",), ("add_side", 0)])
    side = np.random.default_rng(44).standard_normal((1, n, m)).astype(np.float32)
    plan = K.plan_spmm(sw, n, program=prog, bias=bias)
    want = oracle.spmm_exec(sw, x, prog, bias, sides=side)
    rc, got, _ = _host_abi_call(plan, x, "kn", sides=side, chunk=1536)
    assert rc == 0
    check_equal(got, want, prog, "si_spmm_host sides")
    got2 = K.spmm_exec_host(plan, x, layout="kn", chunk=1024, sides=side).numpy()
    check_equal(got2, want, prog, "spmm_exec_host sides")
    with pytest.raises(ValueError):
        K.spmm_exec_host(plan, x, layout="kn")


def test_spmm_exec_host_out_array():
    """spmm_exec(out=<numpy array>) as the reference's signature allows
    (spmm.py:306-309): filled in place and returned; a wrong dtype raises."""
    w, x, bias, scales = baseline_inputs(512, 256, 1000, 0.8, 45)
    sw = P.encode_sparse(w, scales)
    prog = workloads.program("requant_u8", scales)
    plan = K.plan_spmm(sw, 1000, program=prog, bias=bias)
    out = np.zeros((1000, 512), np.uint8)
    res = K.spmm_exec(plan, K.relayout_activation(x), out=out)
    assert res is out
    check_equal(out, oracle.spmm_exec(sw, x, prog, bias), prog, "host out")
    with pytest.raises(ValueError):
        K.spmm_exec(plan, K.relayout_activation(x), out=np.zeros((1000, 512), np.int32))


def test_host_entry_concurrent_threads():
    """Reentrancy: two threads run spmm_exec_host on different
    plans and inputs at once, each with its own workspace and copy streams;
    both results are exact."""
    import threading
    cases = []
    for seed, (m, k, n) in ((51, (1024, 1024, 12000)), (52, (768, 2048, 9000))):
        w, x, bias, scales = baseline_inputs(m, k, n, 0.9, seed)
        sw = P.encode_sparse(w, scales)
        prog = workloads.program("requant_u8", scales)
        plan = K.plan_spmm(sw, n, program=prog, bias=bias)
        cases.append((plan, torch.from_numpy(x).pin_memory(), oracle.spmm_exec(sw, x, prog, bias), prog))
    results = [None, None]
    errors = []

    def worker(i):
        try:
            torch.cuda.set_device(0)
            with torch.cuda.stream(torch.cuda.Stream()):
                for _ in range(3):
                    results[i] = K.spmm_exec_host(cases[i][0], cases[i][1], layout="kn", chunk=2048).numpy()
        except Exception as ex:  # surfaced below
            errors.append(ex)

    th = [threading.Thread(target=worker, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    for i in range(2):
        check_equal(results[i], cases[i][2], cases[i][3], ("thread", i))


@pytest.mark.parametrize("kernel", ["auto", "gather", "tc", "sp"])
@pytest.mark.parametrize("col0", [0, 16, 3])
def test_output_into_wider_buffer(kernel, col0):
    """out may be a column block of a wider [N, ldo] buffer (ldo > M, base
    offset col0): the row-shard write path (parallel.RowShardedSpmm).  A
    16-byte-aligned block takes the TMA-store epilogue, col0 = 3 the direct
    stores; the columns around the block stay untouched."""
    m, k, n = 1024, 1024, 1000
    w, x, bias, scales = baseline_inputs(m, k, n, 0.9, 71)
    sw = P.encode_sparse(w, scales)
    prog = workloads.program("requant_u8", scales)
    plan = K.plan_spmm(sw, n, program=prog, bias=bias)
    act = K.relayout_tokens(np.ascontiguousarray(x.T))
    wide = torch.full((n, m + 48), 0x5A, dtype=torch.uint8, device="cuda")
    view = wide[:, col0: col0 + m]
    K.spmm_exec(plan, act, out=view, kernel=kernel)
    got = wide.cpu().numpy()
    check_equal(got[:, col0: col0 + m], oracle.spmm_exec(sw, x, prog, bias), prog, (kernel, col0))
    assert (got[:, :col0] == 0x5A).all() and (got[:, col0 + m:] == 0x5A).all()


@pytest.mark.parametrize("m,k,n,ratio,kind", [
    (256, 1280, 100, 0.0, "gelu_erf_u8"),   # largest staged slab; 320 tiles per group: staged tiles + L2 tail
    (64, 1296, 48, 0.5, "s32"),             # one row past the slab limit: direct loads
    (768, 768, 128, 0.9, "deq_f32"),        # BASELINE config 1's shape (the cell AUTO sends to K1s)
    (36, 1008, 528, 0.9, "requant_u8"),     # ragged tokens over several token tiles
    (4, 16, 17, 0.0, "s32"),                # one group, one 16-byte chunk
])
def test_staged_gather_kernel(m, k, n, ratio, kind):
    """K1s (spmm_gather.cu): the gather kernel with the activation slab and
    each warp's micro-tiles staged in shared memory by cp.async, against the
    oracle, through kernel="gather" and through AUTO, both layouts."""
    w, x, bias, scales = baseline_inputs(m, k, n, ratio, 4321 + m + k)
    sw = P.encode_sparse(w, scales)
    prog = workloads.program(kind, scales, a_zp=3)
    want = oracle.spmm_exec(sw, x, prog, bias)
    for kernel in ("gather", "auto"):
        for layout in ("kn", "nk"):
            check_equal(run(sw, x, prog, bias, kernel=kernel, layout=layout), want, prog, (m, k, n, kernel, layout))
