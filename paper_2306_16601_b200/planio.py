"""On-disk container for execution plans: the packed weight, its epilogue
program and the device plan image, so a deployment loads a linear without
re-encoding or re-packing (the reference's SPEC
describes such a container as its model-io module).

Layout (little-endian, byte-deterministic for identical plans):

    magic  b"SI4P"                      4 bytes
    version u32                         4 bytes
    meta_len u64                        8 bytes
    meta   UTF-8 JSON (meta_len bytes): scalars + a blob table
           {name: [offset, length, dtype, shape]} with offsets relative to
           the blob section
    blobs  each 64-byte aligned, in table order

The plan image (csrc/image.h) is position independent, so it is stored as
is and uploaded on load; the host arrays are kept so the loaded plan is a
complete ``SpmmPlan`` (oracle checks, re-planning for another N).
"""

from __future__ import annotations

import json
import struct

import numpy as np
import torch

from .kernels.epilogue import EpilogueProgram
from .kernels.spmm import SpmmPlan, _device, partition_tasks, plan_info
from .sparse import Sparse4x1Weight
from .tensor import DType

MAGIC = b"SI4P"
VERSION = 1
_ALIGN = 64


class PlanFormatError(ValueError):
    """Malformed plan container (bad magic, version, bounds, lengths)."""


def _blobs(plan: SpmmPlan) -> dict:
    sw, p = plan.weight, plan.program
    return {
        "group_ptr": sw.group_ptr, "idx": sw.idx, "vals": sw.vals, "nnz": sw.nnz, "scales": sw.scales,
        "bias": plan.bias, "scale_in": p.scale_in, "ops": p.ops, "fparams": p.fparams, "iparams": p.iparams,
        "luts": p.luts, "chans": p.chans, "image": plan.image,
    }


def save_plan(plan: SpmmPlan, path: str) -> None:
    """Write ``plan`` to ``path`` (see the module docstring for the format)."""
    blobs = _blobs(plan)
    table, payload, off = {}, [], 0
    for name, arr in blobs.items():
        a = np.ascontiguousarray(arr)
        b = a.tobytes()
        pad = (-off) % _ALIGN
        payload.append(b"\0" * pad)
        off += pad
        table[name] = [off, len(b), a.dtype.str, list(a.shape)]
        payload.append(b)
        off += len(b)
    sw, p = plan.weight, plan.program
    meta = {"n": plan.n, "bn": plan.bn, "threads": plan.threads,
            "weight": {"rows": sw.rows, "cols": sw.cols, "logical_rows": sw.logical_rows},
            "program": {"a_zp": p.a_zp, "out_dtype": p.out_dtype.value, "n_sides": p.n_sides},
            "blobs": table}
    mb = json.dumps(meta, sort_keys=True, separators=(",", ":")).encode()
    with open(path, "wb") as f:
        f.write(MAGIC + struct.pack("<IQ", VERSION, len(mb)) + mb)
        head = 16 + len(mb)
        f.write(b"\0" * ((-head) % _ALIGN))
        for chunk in payload:
            f.write(chunk)


def load_plan(path: str, device=None) -> SpmmPlan:
    """Read a container written by save_plan and upload its image."""
    with open(path, "rb") as f:
        data = f.read()
    if len(data) < 16 or data[:4] != MAGIC:
        raise PlanFormatError("not a plan container (bad magic)")
    version, mlen = struct.unpack("<IQ", data[4:16])
    if version != VERSION:
        raise PlanFormatError(f"plan container version {version} (expected {VERSION})")
    if 16 + mlen > len(data):
        raise PlanFormatError("truncated metadata")
    try:
        meta = json.loads(data[16:16 + mlen].decode())
    except (UnicodeDecodeError, json.JSONDecodeError) as ex:
        raise PlanFormatError(f"bad metadata: {ex}") from None
    base = 16 + mlen
    base += (-base) % _ALIGN
    arrs = {}
    try:
        for name, (off, length, dt, shape) in meta["blobs"].items():
            if off < 0 or length < 0 or base + off + length > len(data):
                raise PlanFormatError(f"blob {name} out of bounds")
            dtype = np.dtype(dt)
            if int(np.prod(shape, dtype=np.int64)) * dtype.itemsize != length:
                raise PlanFormatError(f"blob {name}: length does not match its shape")
            arrs[name] = np.frombuffer(data, dtype=dtype, count=length // dtype.itemsize,
                                       offset=base + off).reshape(shape).copy()
        w, pm = meta["weight"], meta["program"]
        sw = Sparse4x1Weight(rows=w["rows"], cols=w["cols"], logical_rows=w["logical_rows"],
                             group_ptr=arrs["group_ptr"], idx=arrs["idx"], vals=arrs["vals"], nnz=arrs["nnz"],
                             scales=arrs["scales"])
        prog = EpilogueProgram(scale_in=arrs["scale_in"], a_zp=pm["a_zp"], ops=arrs["ops"], fparams=arrs["fparams"],
                               iparams=arrs["iparams"], luts=arrs["luts"], chans=arrs["chans"],
                               out_dtype=DType(pm["out_dtype"]), n_sides=pm["n_sides"])
        n, bn, threads = int(meta["n"]), int(meta["bn"]), int(meta["threads"])
    except KeyError as ex:
        raise PlanFormatError(f"missing field {ex}") from None
    image = np.ascontiguousarray(arrs["image"], dtype=np.uint8)
    if image.ndim != 1:
        raise PlanFormatError("plan image must be a byte vector")
    # native structural check before anything reads the header: size, magic,
    # header consistency, every section inside the image
    from . import _lib
    if _lib.lib().si_plan_image_validate(_lib.ptr(image), image.nbytes) != 0:
        raise PlanFormatError("bad plan image: " + _lib.lib().si_last_error().decode(errors="replace"))
    info = plan_info(image)
    if info["m"] != sw.logical_rows or info["k"] != sw.cols or info["groups"] != sw.groups \
            or info["padded_blocks"] != int(sw.group_ptr[-1]):
        raise PlanFormatError("plan image does not match the packed weight")
    if info["out_dtype"] != {"f32": 0, "s8": 1, "u8": 2, "s32": 3}[prog.out_dtype.value]:
        raise PlanFormatError("plan image does not match the program")
    image_dev = torch.from_numpy(image).to(_device(device))
    return SpmmPlan(weight=sw, n=n, bn=bn, num_bn=-(-n // bn), threads=threads,
                    tasks=partition_tasks(sw.groups, -(-n // bn), threads), comp=sw.row_sums(), bias=arrs["bias"],
                    program=prog, image=image, image_dev=image_dev, info=info)
