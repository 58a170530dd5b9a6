"""CPU-side checks of the C-ABI library: it loads, exports every symbol that
include/dit.h declares, and its host-only entry points behave."""
import ctypes as C
import os
import re

import pytest

import synth
from paper_2604_08123_b200 import dit

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "dit.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(?:int|void|size_t|double|const char\*)\s+\**\s*(\w+)\s*\(", src)
    return sorted(set(names))


def test_library_exports_every_declared_symbol():
    lib = dit.load_library()
    names = header_functions()
    assert "dit_step" in names and "lora_register" in names and "controlnet_inject" in names and "sp_init" in names
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # and the binding covers them all, with the same names
    assert set(names) <= set(dit.EXPORTS), set(names) - set(dit.EXPORTS)


def test_workspace_bytes_host_only():
    lib = dit.load_library()
    c = dit.make_config(synth.TINY, 2, 16, 8, 4, 1)
    n = lib.dit_workspace_bytes(C.byref(c))
    assert n > 0
    big = dit.make_config(synth.FLUX, 8, 4096, 512, 64, 4)
    nb = lib.dit_workspace_bytes(C.byref(big))
    # activations for B=8 x 4608 rows + 4 adapter slots of ~448 MB: a few GB, well under 180 GB
    assert 3e9 < nb < 20e9, nb
    b16 = dit.make_config(synth.TINY, 16, 16, 8)          # B_max = 16 (e.g. 8 CFG requests)
    assert lib.dit_workspace_bytes(C.byref(b16)) > n
    bad = dit.make_config(synth.TINY, 17, 16, 8)          # B_max > 16
    assert lib.dit_workspace_bytes(C.byref(bad)) == 0
    # a single-GPU workspace drops the SP all-to-all buffers: 16 B_max N D bytes (1.8 GB here)
    one = dit.make_config(synth.FLUX, 8, 4096, 512, 64, 4, max_sp_world=1)
    n1 = lib.dit_workspace_bytes(C.byref(one))
    assert nb - n1 == 16 * 8 * 4608 * 3072 - 65536, nb - n1
    badsp = dit.make_config(synth.TINY, 2, 16, 8, max_sp_world=65)
    assert lib.dit_workspace_bytes(C.byref(badsp)) == 0
    bad2 = dit.make_config(synth.TINY, 2, 16, 8)
    bad2.rope_axes[0] = 6                                   # axes no longer sum to head dim
    assert lib.dit_workspace_bytes(C.byref(bad2)) == 0


def test_create_rejects_bad_arguments_before_touching_the_device():
    lib = dit.load_library()
    c = dit.make_config(synth.TINY, 2, 16, 8)
    ctx = C.c_void_p()
    assert lib.dit_create(C.byref(c), 0, None, 0, C.byref(ctx)) == dit.CODES["DIT_EINVAL"]
    assert b"workspace" in lib.dit_last_error(None)
    assert lib.dit_create(C.byref(c), 0, C.c_void_p(256), 16, C.byref(ctx)) == dit.CODES["DIT_ENOMEM"]
    assert not ctx.value
