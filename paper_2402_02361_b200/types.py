"""ctypes mirrors of include/tt/tt_types.h plus problem builders.

The builders reproduce the reference's fixtures and the benchmark subgraphs
(proj/tests/test_helpers.hpp:16-101) so the parity
tests read like the reference's own tests. Axis ids: spatial axes first in
op order, then reduction axes.
"""
from __future__ import annotations

import ctypes as C

TT_MAX_AXES = 8
TT_MAX_BUFFERS = 6
TT_MAX_UNROLL = 4
TT_IO_INPUT, TT_IO_OUTPUT = 0, 1
TT_OP_TILED, TT_OP_ELEMENTWISE = 0, 1
TT_STMT_WIDTH, TT_BLOCK_WIDTH = 24, 23
TT_TOGGLE_COMPUTE, TT_TOGGLE_MEMORY, TT_TOGGLES_ALL = 1, 2, 3


class DeviceSpec(C.Structure):
    """tiletune::DeviceSpec (device.hpp:29-39)."""

    _fields_ = [("m_l0", C.c_int64), ("m_l1", C.c_int64), ("pu_l1", C.c_int64),
                ("n_l1", C.c_int64), ("pu_l2", C.c_int64), ("n_l2", C.c_int64),
                ("t_p", C.c_double), ("t_m", C.c_double), ("element_bytes", C.c_int64)]


class OracleSpec(C.Structure):
    """tiletune::OracleDevice (oracle.hpp:40-47)."""

    _fields_ = [("hidden", DeviceSpec), ("stride_coeff", C.c_double), ("occupancy_coeff", C.c_double),
                ("launch_overhead_s", C.c_double), ("noise_sigma", C.c_double), ("seed", C.c_uint64)]


class BufferSpec(C.Structure):
    _fields_ = [("io", C.c_int32), ("n_axes", C.c_int32), ("axes", C.c_int32 * TT_MAX_AXES)]


class OpSpec(C.Structure):
    """tiletune::TensorOpSpec (workload.hpp:47-57) with axis ids."""

    _fields_ = [("n_spatial", C.c_int32), ("n_reduction", C.c_int32),
                ("extent", C.c_int64 * TT_MAX_AXES), ("n_buffers", C.c_int32),
                ("fused_elementwise", C.c_int32), ("kind", C.c_int32), ("_pad", C.c_int32),
                ("buffers", BufferSpec * TT_MAX_BUFFERS)]

    @property
    def n_inputs(self) -> int:
        return sum(1 for b in range(self.n_buffers) if self.buffers[b].io == TT_IO_INPUT)

    @property
    def n_statements(self) -> int:
        return 2 * self.n_inputs + 2

    @property
    def n_blocks(self) -> int:
        return 1 if self.kind == TT_OP_ELEMENTWISE else 3 * self.n_inputs + 2


class Sketch(C.Structure):
    """tiletune::Sketch as generate_sketch(op, true) builds it (schedule.cpp:150-164)."""

    _fields_ = [("op", OpSpec), ("n_unroll", C.c_int32), ("_pad", C.c_int32),
                ("unroll", C.c_int64 * TT_MAX_UNROLL)]

    @property
    def cols(self) -> int:
        return 4 * self.op.n_spatial + 3 * self.op.n_reduction + 1


def make_op(spatial, reduction, buffers, fused=0, kind=None) -> OpSpec:
    """spatial/reduction: lists of (name, extent); buffers: (axis names, io)."""
    op = OpSpec()
    names = [n for n, _ in spatial] + [n for n, _ in reduction]
    op.n_spatial, op.n_reduction = len(spatial), len(reduction)
    for i, (_, e) in enumerate(list(spatial) + list(reduction)):
        op.extent[i] = int(e)
    op.n_buffers = len(buffers)
    for b, (axes, io) in enumerate(buffers):
        op.buffers[b].io = io
        op.buffers[b].n_axes = len(axes)
        for q, a in enumerate(axes):
            op.buffers[b].axes[q] = names.index(a)
    op.fused_elementwise = fused
    op.kind = (TT_OP_TILED if reduction else TT_OP_ELEMENTWISE) if kind is None else kind
    return op


def make_gemm(m, n, k, fused=0) -> OpSpec:
    """test_helpers.hpp:66-78."""
    return make_op([("m", m), ("n", n)], [("k", k)],
                   [(["m", "k"], TT_IO_INPUT), (["k", "n"], TT_IO_INPUT),
                    (["m", "n"], TT_IO_OUTPUT)], fused)


def make_conv(f, y, x, c, r) -> OpSpec:
    """test_helpers.hpp:89-101: spatial (f, y, x), reduction (c, r)."""
    return make_op([("f", f), ("y", y), ("x", x)], [("c", c), ("r", r)],
                   [(["c", "y", "x"], TT_IO_INPUT), (["f", "c", "r"], TT_IO_INPUT),
                    (["f", "y", "x"], TT_IO_OUTPUT)])


def make_bmm(b, m, n, k) -> OpSpec:
    """BERT batch-matmul: A[b,m,k] B[b,k,n] C[b,m,n]."""
    return make_op([("b", b), ("m", m), ("n", n)], [("k", k)],
                   [(["b", "m", "k"], TT_IO_INPUT), (["b", "k", "n"], TT_IO_INPUT),
                    (["b", "m", "n"], TT_IO_OUTPUT)])


def make_elementwise(h, w) -> OpSpec:
    """test_helpers.hpp:80-87."""
    return make_op([("h", h), ("w", w)], [],
                   [(["h", "w"], TT_IO_INPUT), (["h", "w"], TT_IO_OUTPUT)],
                   kind=TT_OP_ELEMENTWISE)


def make_sketch(op: OpSpec, unroll=(1, 4, 16)) -> Sketch:
    sk = Sketch()
    sk.op = op
    sk.n_unroll = len(unroll)
    for i, u in enumerate(unroll):
        sk.unroll[i] = u
    return sk


def reference_device() -> DeviceSpec:
    """proj/samples/device.txt == test_helpers.hpp:16-28."""
    return DeviceSpec(256, 4096, 4, 32, 8, 32, 1.0e12, 1.0e11, 4)


def oracle_a() -> "OracleSpec":
    """test_helpers.hpp:30-45 == proj/samples/oracle_a.txt."""
    return OracleSpec(DeviceSpec(192, 3072, 4, 32, 6, 16, 8.0e11, 1.2e11, 4), 0.35, 1.5, 2.0e-6, 0.03, 90001)


def oracle_b() -> "OracleSpec":
    """test_helpers.hpp:47-64 == proj/samples/oracle_b.txt."""
    return OracleSpec(DeviceSpec(128, 6144, 2, 64, 12, 64, 1.5e12, 0.9e11, 4), 0.5, 2.0, 1.0e-6, 0.03, 90002)


def hash_str(s: str) -> int:
    """FNV-1a (common.hpp:74-82)."""
    h = 1469598103934665603
    for ch in s.encode():
        h = ((h ^ ch) * 1099511628211) & M64
    return h


def oracle_b_hidden() -> DeviceSpec:
    """proj/samples/oracle_b.txt hidden device (test_helpers.hpp:47-64)."""
    return DeviceSpec(128, 6144, 2, 64, 12, 64, 1.5e12, 0.9e11, 4)


# The subgraphs of BASELINE.json's configs.
WORKLOADS = {
    "gemm1024": lambda: make_gemm(1024, 1024, 1024),
    "r50_stem": lambda: make_conv(64, 112, 112, 3, 49),
    "r50_c1x1_64": lambda: make_conv(64, 56, 56, 64, 1),
    "r50_c3x3_64": lambda: make_conv(64, 56, 56, 64, 9),
    "r50_c1x1_256": lambda: make_conv(256, 56, 56, 64, 1),
    "r50_c3x3_128": lambda: make_conv(128, 28, 28, 128, 9),
    "r50_c3x3_256": lambda: make_conv(256, 14, 14, 256, 9),
    "r50_c3x3_512": lambda: make_conv(512, 7, 7, 512, 9),
    "bert_qkv": lambda: make_gemm(128, 2304, 768),
    "bert_proj": lambda: make_gemm(128, 768, 768),
    "bert_ffn1": lambda: make_gemm(128, 3072, 768),
    "bert_ffn2": lambda: make_gemm(128, 768, 3072),
    "bert_bmm_qk": lambda: make_bmm(12, 128, 128, 64),
    "bert_bmm_pv": lambda: make_bmm(12, 128, 64, 128),
}


GOLDEN = 0x9E3779B97F4A7C15
M64 = (1 << 64) - 1


def _scramble64(x: int) -> int:
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


def mix64(x: int) -> int:
    """common.hpp:52-57."""
    return _scramble64((x + GOLDEN) & M64)


def derive_seed(base: int, *tags: int) -> int:
    """common.hpp:66-72."""
    for a in tags:
        base = mix64(base ^ mix64(a))
    return base


TAG_INIT = 0x696E6974  # tuner.cpp:139-140 "init"
