"""CPU-side checks of the C-ABI boundary: libgem.so builds for sm_100a, loads
without a GPU, exports every symbol include/gem.h declares, and its ctypes
struct layouts match the C header.  No compute calls (no GPU here)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def libgem():
    from paper_2509_25075_b200 import build
    build.build()
    from paper_2509_25075_b200 import binding
    return binding


def test_exports_every_header_symbol(libgem):
    names = libgem.header_symbols()
    assert len(names) >= 12 and {"gem_init", "gem_forward", "gem_backward", "gem_step", "gem_render_volume"} <= set(names)
    out = subprocess.run(["nm", "-D", "--defined-only", libgem.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (gem_\w+)", out))
    assert set(names) <= exported, set(names) - exported
    L = libgem.lib()
    for n in names:
        assert getattr(L, n) is not None


def test_status_strings_host_only(libgem):
    assert libgem.status_string(0) == "ok"
    assert "capacity" in libgem.status_string(libgem.GEM_E_CAPACITY)


def test_struct_layouts_match_header(libgem, tmp_path):
    src = tmp_path / "sz.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "gem.h"\nint main(){'
                   'printf("%zu %zu %zu %zu %zu %zu %zu\\n", sizeof(gem_config), sizeof(gem_soa), sizeof(gem_batch),'
                   ' sizeof(gem_stats_t), offsetof(gem_config, list_capacity), offsetof(gem_config, flags),'
                   ' offsetof(gem_batch, observed)); return 0;}\n')
    exe = tmp_path / "sz"
    subprocess.check_call(["gcc", "-I" + os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    vals = [int(x) for x in subprocess.check_output([str(exe)]).split()]
    b = libgem
    assert vals == [ctypes.sizeof(b.GemConfigC), ctypes.sizeof(b.GemSoaC), ctypes.sizeof(b.GemBatchC),
                    ctypes.sizeof(b.GemStatsC), b.GemConfigC.list_capacity.offset, b.GemConfigC.flags.offset,
                    b.GemBatchC.observed.offset]


def test_sass_is_sm100a(libgem):
    out = subprocess.run(["cuobjdump", "--list-elf", libgem.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_product_path_never_touches_oracle():
    pkg = os.path.join(ROOT, "paper_2509_25075_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle", txt, re.M), f
                assert "gem_oracle" not in txt and "liboracle" not in txt, f


def test_binding_fails_loudly_without_library(monkeypatch):
    from paper_2509_25075_b200 import binding
    monkeypatch.setattr(binding, "_lib", None)
    monkeypatch.setattr(binding, "LIB_PATH", "/nonexistent/libgem.so")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        binding.lib()
