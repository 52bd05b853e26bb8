"""The drop-in boundary without a GPU: the sm_100a library loads, exports
every entry point include/tt/tt.h declares (and the ctypes binding binds
exactly those), its host-side problem-model functions agree with the
oracle, and compute entry points fail loudly (E_CUDA) instead of falling
back to the CPU when no device is usable.
"""
import ctypes as C
import os
import re
import subprocess

import pytest
import torch

from paper_2402_02361_b200 import _capi
from paper_2402_02361_b200.types import (WORKLOADS, DeviceSpec, Sketch, make_elementwise, make_gemm, make_op,
                                         make_sketch, reference_device, TT_IO_INPUT, TT_IO_OUTPUT)
from tests import _refs as R

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tt", "tt.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tt_[a-z0-9_]+)\s*\(", src)))


def test_header_and_binding_agree():
    assert declared() == sorted(_capi.EXPORTED)


def test_library_exports_every_declared_symbol():
    assert os.path.exists(_capi.LIB_PATH), "build first: python -m paper_2402_02361_b200.build"
    out = subprocess.run(["nm", "-D", "--defined-only", _capi.LIB_PATH], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = [s for s in declared() if s not in exported]
    assert not missing, missing
    _capi.lib()  # binds every signature


def test_library_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _capi.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_status_codes_mirror_reference():
    L = _capi.lib()
    names = [L.tt_status_code(i).decode() for i in range(8)]
    assert names[1:6] == ["E_PARSE", "E_VALIDATE", "E_CONFIG", "E_STATE", "E_IO"]
    assert names[6] == "E_CUDA"


def test_sketch_space_draws_match_oracle():
    L = _capi.lib()
    for name in ["gemm1024", "r50_stem", "r50_c3x3_512", "bert_qkv", "bert_bmm_pv"]:
        op = WORKLOADS[name]()
        sk = Sketch()
        assert L.tt_sketch_from_op(C.byref(op), 1, C.byref(sk)) == 0
        ref = make_sketch(op)
        assert bytes(sk) == bytes(ref)
        assert L.tt_space_size(C.byref(sk)) == R.oracle().tto_space_size(C.byref(ref))
        assert L.tt_draws_per_schedule(C.byref(sk)) == R.oracle().tto_draws_per_schedule(C.byref(ref))


def test_sketch_validation_errors():
    L = _capi.lib()
    sk = Sketch()
    bad = make_gemm(0, 8, 8)
    assert _capi.lib().tt_status_code(L.tt_sketch_from_op(C.byref(bad), 1, C.byref(sk))).decode() == "E_VALIDATE"
    # buffer referencing a missing axis
    op = make_op([("m", 8)], [("k", 8)], [(["m", "k"], TT_IO_INPUT), (["m"], TT_IO_OUTPUT)])
    op.buffers[0].axes[1] = 7
    assert L.tt_sketch_from_op(C.byref(op), 1, C.byref(sk)) != 0
    ew = make_elementwise(64, 48)
    assert L.tt_sketch_from_op(C.byref(ew), 1, C.byref(sk)) == 0 and sk.op.kind == 1


def test_device_validation():
    L = _capi.lib()
    assert L.tt_validate_device(C.byref(reference_device())) == 0
    d = reference_device()
    d.n_l1 = 24  # not a power of two (device.cpp:105-108)
    assert L.tt_status_code(L.tt_validate_device(C.byref(d))).decode() == "E_VALIDATE"
    d = reference_device()
    d.t_p = 0.0
    assert L.tt_validate_device(C.byref(d)) != 0


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback_without_gpu():
    from paper_2402_02361_b200 import tiletune as tt
    with pytest.raises(tt.TTError) as e:
        tt.Context(0)
    assert e.value.code == "E_CUDA"
    h = C.c_void_p()
    assert _capi.lib().tt_ctx_create(0, C.byref(h)) == 6


def test_struct_layouts_match_header():
    # tt_types.h POD sizes as the C compiler lays them out
    src = ('#include "tt/tt_types.h"\n#include "tt/tt.h"\n#include <stdio.h>\n'
           'int main(){printf("%zu %zu %zu %zu %zu\\n", sizeof(tt_device_spec), sizeof(tt_op_spec),'
           ' sizeof(tt_sketch), sizeof(tt_round_config), sizeof(tt_round_result));}')
    d = os.path.join(ROOT, "oracle", "_build")
    os.makedirs(d, exist_ok=True)
    c, exe = os.path.join(d, "layout.c"), os.path.join(d, "layout")
    open(c, "w").write(src)
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe], check=True)
    got = [int(x) for x in subprocess.run([exe], capture_output=True, text=True).stdout.split()]
    want = [C.sizeof(DeviceSpec), C.sizeof(make_gemm(1, 1, 1)), C.sizeof(Sketch), C.sizeof(_capi.RoundConfig),
            C.sizeof(_capi.RoundResult)]
    assert got == want


def test_magic_round_up_is_exact():
    """The L1/L2 round-ups of the 32-bit draft-cost mode (tt_device.cuh
    ceil_div_magic): q = umulhi(floor((2^64 - 1) / b) + 1, a) is floor(a / b)
    for every a < 2^32 and b < 2^32 (Lemire, Kaser, Kurz 2019), and
    q + (q * b != a) the round-up draft.cpp:108-127 takes with int64
    division. Checked here on the formula: every b up to 4,096 and random
    large b, against exact integer arithmetic at the edges and on random a."""
    import random
    rnd = random.Random(7)
    bs = list(range(2, 4097)) + [rnd.randrange(4097, 1 << 32) for _ in range(2000)] + [(1 << 32) - 1]
    for b in bs:
        m = (2 ** 64 - 1) // b + 1
        for a in [0, 1, b - 1, b, b + 1, (1 << 32) - 1, (1 << 32) - b, ((1 << 32) - 1) // b * b] + \
                 [rnd.randrange(0, 1 << 32) for _ in range(8)]:
            q = (m * a) >> 64
            assert q == a // b
            assert q + (q * b != a) == -(-a // b)
