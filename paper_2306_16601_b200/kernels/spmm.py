"""INT8 4x1-block sparse weight x dense u8 activation GEMM on B200.

Drop-in mirror of the reference's ``sparseinfer.kernels.spmm``
(/root/reference/pkg/src/sparseinfer/kernels/spmm.py): same names, argument
meaning, validation order and exception types.  What changes is underneath:

* ``plan_spmm`` (spmm.py:160-189) builds a *plan image* in the native
  library (csrc/plan.cpp): GPU tile formats of the weight, the compensation
  adj[m] = bias[m] - a_zp*comp[m], and the compiled epilogue.  The image is
  uploaded once to HBM and cached on the plan.
* ``relayout_activation`` / ``relayout_tokens`` (spmm.py:82-107) do not
  relayout: the kernels read [K, N] and token-major [N, K] directly, so the
  returned ``ActivationLayout`` just wraps the CUDA tensor and its
  orientation.  ``data`` is therefore the activation itself, not the
  [NUM_BN, K, BN] panel stack.
* ``spmm_exec`` (spmm.py:283-333) launches on ``torch.cuda.current_stream()``
  and returns a CUDA tensor [N, M] of the program's dtype; ``pool`` is
  accepted and ignored (the GPU grid replaces the CPU task pool).
* ``spmm_ref`` (spmm.py:401-427) is a naive one-thread-per-output kernel
  with the interpreted epilogue -- an independent device implementation of
  the same contract, not the CPU oracle (that lives in oracle/ and is test
  infrastructure).

PyTorch is used only for device memory and streams.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from .. import _lib
from ..sparse import Sparse4x1Weight
from ..tensor import DType
from .epilogue import EpilogueProgram, build_program

DEFAULT_BN = 64

_TORCH_DT = {DType.F32: torch.float32, DType.S8: torch.int8, DType.U8: torch.uint8,
             DType.S32: torch.int32}


def raw_program(sw: Sparse4x1Weight, a_zp: int = 0) -> EpilogueProgram:
    """Epilogue emitting the wrapped S32 accumulator (spmm.py:35-37)."""
    return build_program(sw.scales, 1.0, a_zp, None)


def _ld(t: torch.Tensor) -> int:
    """Row pitch in elements; a single-row tensor may carry any stride(0)."""
    return int(t.shape[1]) if t.shape[0] == 1 else int(t.stride(0))


def _device(device=None) -> torch.device:
    if device is not None:
        return torch.device(device)
    if not torch.cuda.is_available():
        raise RuntimeError("sparseinfer_b200 needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _to_cuda_u8(a, device=None) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        if a.dtype != torch.uint8:
            a = a.to(torch.uint8)
        t = a if a.is_cuda else a.to(_device(device), non_blocking=a.is_pinned())
    else:
        arr = np.ascontiguousarray(a, dtype=np.uint8)
        t = torch.from_numpy(arr).to(_device(device))
    return t if t.is_contiguous() else t.contiguous()


@dataclass(frozen=True)
class ActivationLayout:
    """A u8 activation resident on the GPU, [K, N] ("kn") or [N, K] ("nk").

    Mirrors spmm.py:40-51; ``bn`` is kept for plan matching only."""

    data: torch.Tensor
    k: int
    n: int
    bn: int
    orient: str = "kn"

    @property
    def num_bn(self) -> int:
        return -(-self.n // self.bn)

    @property
    def ld(self) -> int:
        return _ld(self.data)


def relayout_activation(a, bn: int = DEFAULT_BN, out=None, device=None) -> ActivationLayout:
    """Wrap a [K, N] u8 activation (spmm.py:82-93); copies to the GPU if needed."""
    t = _to_cuda_u8(a, device)
    if t.ndim != 2:
        raise ValueError("activation must be 2-D [K, N]")
    k, n = t.shape
    if n == 0:
        raise ValueError("N must be positive")
    if out is not None:
        out.copy_(t)
        t = out
    return ActivationLayout(t, int(k), int(n), bn, "kn")


def relayout_tokens(x, bn: int = DEFAULT_BN, out=None, device=None) -> ActivationLayout:
    """Wrap a token-major [N, K] u8 activation (spmm.py:96-107)."""
    t = _to_cuda_u8(x, device)
    if t.ndim != 2:
        raise ValueError("activation must be 2-D [N, K]")
    n, k = t.shape
    if n == 0:
        raise ValueError("N must be positive")
    if out is not None:
        out.copy_(t)
        t = out
    return ActivationLayout(t, int(k), int(n), bn, "nk")


@dataclass(frozen=True)
class SpmmPlan:
    """Immutable plan for one sparse linear layer (spmm.py:110-133), plus the
    native plan image (host bytes and its HBM copy)."""

    weight: Sparse4x1Weight
    n: int
    bn: int
    num_bn: int
    threads: int
    tasks: tuple
    comp: np.ndarray
    bias: np.ndarray
    program: EpilogueProgram
    image: np.ndarray = field(repr=False, default=None)
    image_dev: torch.Tensor = field(repr=False, default=None)
    info: dict = field(default_factory=dict)

    m_block = 4
    k_block = 4

    @property
    def n_block(self) -> int:
        return self.bn

    @property
    def m(self) -> int:
        return self.weight.logical_rows


def partition_tasks(groups: int, num_bn: int, threads: int) -> tuple:
    """The reference's disjoint (group-range, panel-range) cover
    (spmm.py:136-157), kept for API compatibility; the GPU grid does not use it."""

    def split(total, parts):
        parts = max(1, min(parts, total))
        base, rem = divmod(total, parts)
        bounds = np.concatenate([[0], np.cumsum([base + (i < rem) for i in range(parts)])])
        return list(zip(bounds[:-1].tolist(), bounds[1:].tolist()))

    if num_bn >= threads:
        return tuple((0, groups, b0, b1) for b0, b1 in split(num_bn, threads))
    granges = split(groups, max(1, threads // num_bn))
    return tuple((g0, g1, b0, b1) for b0, b1 in split(num_bn, num_bn) for g0, g1 in granges)


_EPI_NAMES = {0: "s32", 1: "deq_f32", 2: "requant", 3: "requant_lut", 4: "deq_table", 5: "generic", 6: "deq_side"}


def _build_image(sw: Sparse4x1Weight, program: EpilogueProgram, bias: np.ndarray):
    L = _lib.lib()
    hw, hp = _lib.HostWeight(sw), _lib.HostProgram(program)
    size = ctypes.c_uint64(0)
    _lib.check(L.si_plan_image_size(ctypes.byref(hw.s), ctypes.byref(hp.s), ctypes.byref(size)),
               "plan_spmm")
    image = np.zeros(size.value, dtype=np.uint8)
    _lib.check(L.si_plan_image_build(ctypes.byref(hw.s), ctypes.byref(hp.s), _lib.ptr(bias),
                                     _lib.ptr(image), size.value), "plan_spmm")
    return image, plan_info(image)


def plan_info(image: np.ndarray) -> dict:
    """Header summary of a plan image (si_plan_info_get); raises on an image
    whose magic / version this library does not know."""
    info = _lib.SiPlanInfo()
    _lib.check(_lib.lib().si_plan_info_get(_lib.ptr(image), ctypes.byref(info)), "plan image")
    return {f: getattr(info, f) for f, _ in info._fields_} | {"epilogue": _EPI_NAMES.get(info.epi_mode, "?")}


def plan_spmm(sw: Sparse4x1Weight, n: int, threads: int = 1, program: EpilogueProgram | None = None,
              bias: np.ndarray | None = None, bn: int = DEFAULT_BN, device=None) -> SpmmPlan:
    """Build and upload the execution plan (spmm.py:160-189)."""
    if n <= 0:
        raise ValueError("N must be positive")
    if threads < 1:
        raise ValueError("threads must be >= 1")
    if bn % 16 != 0 or bn < 16:
        raise ValueError("n_block must be a positive multiple of 16")
    if program is None:
        program = raw_program(sw)
    if program.m != sw.logical_rows:
        raise ValueError("program channel count must match weight rows")
    if bias is None:
        bias = np.zeros(sw.logical_rows, dtype=np.int32)
    bias = np.ascontiguousarray(bias, dtype=np.int32)
    if bias.shape != (sw.logical_rows,):
        raise ValueError("bias must be one s32 per logical output row")
    num_bn = -(-n // bn)
    image, info = _build_image(sw, program, bias)
    image_dev = torch.from_numpy(image).to(_device(device))
    return SpmmPlan(weight=sw, n=n, bn=bn, num_bn=num_bn, threads=threads,
                    tasks=partition_tasks(sw.groups, num_bn, threads), comp=sw.row_sums(),
                    bias=bias, program=program, image=image, image_dev=image_dev, info=info)


def _sides_tensor(sides, plan_n, m, n_sides, device):
    if n_sides == 0:
        return None
    if sides is None:
        raise ValueError(f"program needs {n_sides} side inputs")
    t = sides if isinstance(sides, torch.Tensor) else torch.from_numpy(
        np.ascontiguousarray(sides, dtype=np.float32))
    t = t.to(device=device, dtype=torch.float32).contiguous()
    if t.ndim != 3 or t.shape[0] < n_sides or t.shape[1] != plan_n or t.shape[2] != m:
        raise ValueError(f"program needs {n_sides} side inputs")
    return t


def _run(plan: SpmmPlan, x: torch.Tensor, layout: str, n: int, ldx: int, sides, out,
         kernel: str) -> torch.Tensor:
    L = _lib.lib()
    m = plan.weight.logical_rows
    prog = plan.program
    dev = x.device
    sd = _sides_tensor(sides, n, m, prog.n_sides, dev)
    dt = _TORCH_DT[prog.out_dtype]
    if out is None:
        out = torch.empty((n, m), dtype=dt, device=dev)
    elif (tuple(out.shape) != (n, m) or out.dtype != dt or not out.is_cuda
          or (m > 1 and out.stride(1) != 1) or _ld(out) < m):
        raise ValueError("bad output buffer")
    lay = _lib.LAYOUTS[layout]
    kid = _lib.KERNELS[kernel]
    img = _lib.ptr(plan.image)
    ws_bytes = ctypes.c_uint64(0)
    _lib.check(L.si_spmm_workspace_size(img, n, lay, kid, ctypes.byref(ws_bytes)), "spmm_exec")
    ws = torch.empty(int(ws_bytes.value), dtype=torch.uint8, device=dev) if ws_bytes.value else None
    stream = torch.cuda.current_stream(dev).cuda_stream
    rc = L.si_spmm(img, plan.image_dev.data_ptr(), x.data_ptr(), lay, ldx, n,
                   sd.data_ptr() if sd is not None else None, out.data_ptr(), _ld(out),
                   ws.data_ptr() if ws is not None else None, ws_bytes.value, kid, stream)
    _lib.check(rc, "spmm_exec")
    return out


def spmm_exec(plan: SpmmPlan, act: ActivationLayout, pool=None, sides=None, out=None,
              kernel: str = "auto"):
    """Run the fused SpMM on the GPU (spmm.py:283-333).

    Returns a CUDA tensor [N, M].  ``out`` may be a CUDA tensor (written in
    place) or, as in the reference, a host array (numpy / CPU tensor) of shape
    [N, M] and the program's dtype: the result is computed on the GPU and
    copied into it, and ``out`` itself is returned.  ``kernel`` selects
    "auto", "gather" (K1), "tc" (K2), "ref", or one of the opt-in 2:4
    tensor-core kernels "sp" (K3) / "ws" (K4): token-major X, K <= 1024."""
    sw = plan.weight
    if act.k != sw.cols or act.n != plan.n or act.bn != plan.bn:
        raise ValueError("activation layout does not match the plan")
    host_out = out is not None and not (isinstance(out, torch.Tensor) and out.is_cuda)
    if host_out:
        dt = plan.program.out_dtype
        shape_ok = tuple(out.shape) == (plan.n, sw.logical_rows)
        dtype_ok = (out.dtype == dt.np) if isinstance(out, np.ndarray) else (out.dtype == _TORCH_DT[dt])
        if not (shape_ok and dtype_ok):
            raise ValueError("bad output buffer")
        res = _run(plan, act.data, act.orient, act.n, act.ld, sides, None, kernel)
        if isinstance(out, np.ndarray):
            np.copyto(out, res.cpu().numpy())
        else:
            out.copy_(res)
        return out
    return _run(plan, act.data, act.orient, act.n, act.ld, sides, out, kernel)


def _host_sides(sides, n_sides: int, n: int, m: int):
    """The reference's side check (spmm.py:300-304): a host f32 [n_sides, N, M]
    stack (pack_sides form), contiguous for the per-chunk copies."""
    if n_sides == 0:
        return None
    if sides is None:
        raise ValueError(f"program needs {n_sides} side inputs")
    t = sides if isinstance(sides, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(sides, np.float32))
    if t.is_cuda:
        raise ValueError("spmm_exec_host: sides must be host memory")
    t = t.to(torch.float32).contiguous()
    if t.ndim != 3 or t.shape[0] < n_sides or t.shape[1] != n or t.shape[2] != m:
        raise ValueError(f"program needs {n_sides} side inputs")
    return t


def _host_job(plan: SpmmPlan, x, layout: str, out, sides=None):
    sw = plan.weight
    m = sw.logical_rows
    prog = plan.program
    xt = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x))
    if xt.is_cuda or xt.dtype != torch.uint8 or xt.ndim != 2:
        raise ValueError("spmm_exec_host: x must be a host u8 matrix")
    if layout == "kn":
        k, n = xt.shape
    elif layout == "nk":
        n, k = xt.shape
    else:
        raise ValueError("layout must be 'kn' or 'nk'")
    if k != sw.cols or n != plan.n:
        raise ValueError("activation does not match the plan")
    if xt.stride(1) != 1:
        xt = xt.contiguous()
    st = _host_sides(sides, prog.n_sides, n, m)
    dt = _TORCH_DT[prog.out_dtype]
    if out is None:
        out = torch.empty((n, m), dtype=dt).pin_memory()
    elif tuple(out.shape) != (n, m) or out.dtype != dt or out.is_cuda or (m > 1 and out.stride(1) != 1):
        raise ValueError("bad output buffer")
    job = _lib.SiHostJob(_lib.ptr(plan.image), plan.image_dev.data_ptr(), xt.data_ptr(), _lib.LAYOUTS[layout],
                         _ld(xt), n, out.data_ptr(), _ld(out), st.data_ptr() if st is not None else None)
    return job, (xt, st), out


def spmm_exec_host_batch(items, chunk: int = 8192, kernel: str = "auto") -> list:
    """Several independent spmm_exec calls on host buffers as one pipelined
    chunk sequence (si_spmm_host_batch): ``items`` is a list of
    (plan, x, layout, out) or (plan, x, layout, out, sides) with out None for
    a new pinned tensor and sides the host f32 [n_sides, N, M] stack.  The
    copy-in of one job overlaps the copy-out of the previous one.

    Reentrant: every call sizes and allocates its own device workspace (from
    the caching allocator, on the current stream) and the library gives it a
    private pair of copy streams, so threads may call concurrently."""
    L = _lib.lib()
    if not items:
        return []
    built = [_host_job(*it) for it in items]
    jobs = (_lib.SiHostJob * len(built))(*[b[0] for b in built])
    dev = items[0][0].image_dev.device
    need = ctypes.c_uint64(0)
    _lib.check(L.si_spmm_host_batch_workspace_size(jobs, len(built), chunk, ctypes.byref(need)), "spmm_exec_host")
    ws = torch.empty(int(need.value), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    rc = L.si_spmm_host_batch(jobs, len(built), ws.data_ptr(), need.value, chunk, _lib.KERNELS[kernel], stream)
    _lib.check(rc, "spmm_exec_host")
    return [b[2] for b in built]


def spmm_exec_host(plan: SpmmPlan, x, layout: str = "kn", out=None, chunk: int = 8192,
                   kernel: str = "auto", sides=None) -> torch.Tensor:
    """spmm_exec on host buffers (the reference's call takes host arrays,
    spmm.py:283-333): ``x`` is the logical [K, N] (layout "kn") or token-major
    [N, K] ("nk") u8 activation in host memory, ``sides`` the host f32
    [n_sides, N, M] residual stack the program needs, and the result [N, M]
    comes back in host memory (``out`` or a new pinned tensor).  Token chunks
    are pipelined by the library (si_spmm_host): copy-in, kernel and copy-out
    of neighbouring chunks overlap.  Pinned inputs give full overlap."""
    return spmm_exec_host_batch([(plan, x, layout, out, sides)], chunk=chunk, kernel=kernel)[0]


def spmm_ref(sw: Sparse4x1Weight, a, program: EpilogueProgram | None = None, bias=None,
             sides=None) -> torch.Tensor:
    """Naive device oracle (spmm.py:401-427): ``a`` is the logical [K, N] u8
    activation; output [N, M] identical in every bit to ``spmm_exec`` (up to
    the device GELU for f32 outputs)."""
    x = _to_cuda_u8(a)
    if x.ndim != 2 or x.shape[0] != sw.cols:
        raise ValueError(f"activation rows must equal K={sw.cols}")
    if program is None:
        program = raw_program(sw)
    plan = plan_spmm(sw, int(x.shape[1]), program=program, bias=bias, device=x.device)
    return _run(plan, x, "kn", int(x.shape[1]), _ld(x), sides, None, "ref")


def dot4_accum(a4, b4, acc: int) -> int:
    """The 4-wide u8 x s8 dot-product contract (spmm.py:430-439):
    exact products, wrapping 32-bit accumulation.  This is dp4a.u32.s32."""
    total = int(acc)
    for x, y in zip(a4, b4):
        xv, yv = int(x), int(y)
        if not (0 <= xv <= 255 and -128 <= yv <= 127):
            raise ValueError("dot4 operands out of u8/s8 range")
        total += xv * yv
    return int(np.int64(total).astype(np.uint32).view(np.int32))
