"""C-ABI library checks that need no GPU: it builds/loads, exports every symbol include/de.h
declares, struct layouts match, and without a device the product path fails loudly."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "de.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(de_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_1501_06211_b200.build import build
    build()
    from paper_1501_06211_b200 import binding
    return binding.lib()


def test_exports_every_declared_symbol(lib):
    names = _declared()
    assert "de_setup" in names and "de_solve" in names and "de_factor" in names
    for n in names:
        assert hasattr(lib, n), n


def test_binding_names_mirror_abi():
    from paper_1501_06211_b200 import binding
    for n in _declared():
        if n in ("de_last_error",):
            continue
        assert hasattr(binding, n), n


def test_default_options_and_struct_sizes(lib):
    from paper_1501_06211_b200 import binding as B
    o = B.de_default_options()
    assert o.theta == 0.5 and o.lanczos_k == 10 and o.inner_mode == 1 and o.nranks == 1
    assert o.check_every == 8 and o.use_graph == 1
    # layouts must match the C compiler's view of include/de.h
    import subprocess, tempfile
    src = ('#include "de.h"\n#include <stdio.h>\n#include <stddef.h>\nint main(){printf("%zu %zu %zu %zu %zu",'
           'sizeof(de_options_t), sizeof(de_mesh_t), sizeof(de_stats_t), offsetof(de_options_t, nccl_id),'
           'offsetof(de_stats_t, n_cross));printf(" %zu", sizeof(de_oc_params_t));return 0;}')
    with tempfile.TemporaryDirectory() as d:
        open(os.path.join(d, "t.c"), "w").write(src)
        subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), os.path.join(d, "t.c"), "-o",
                               os.path.join(d, "t")])
        got = list(map(int, subprocess.check_output([os.path.join(d, "t")]).split()))
    assert got == [ctypes.sizeof(B.de_options_t), ctypes.sizeof(B.de_mesh_t), ctypes.sizeof(B.de_stats_t),
                   B.de_options_t.nccl_id.offset, B.de_stats_t.n_cross.offset, ctypes.sizeof(B.de_oc_params_t)]


def test_no_cpu_fallback_without_device(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from synthetic import make_config
    from paper_1501_06211_b200 import binding as B
    p = make_config("c1")
    with pytest.raises(B.DEError) as ei:
        B.Solver.from_problem(p)
    assert ei.value.status in (B.DE_ECUDA,)


def test_invalid_arguments_rejected_before_device(lib):
    from synthetic import make_config
    from paper_1501_06211_b200 import binding as B
    p = make_config("c1")
    with pytest.raises(B.DEError) as ei:   # partition does not divide the mesh
        B.de_setup(2, (32, 16), 1.0, p.fixed, p.density, 1.0, 1e-9, 3.0, 0.3, (5, 8))
    assert ei.value.status == B.DE_EINVAL
    with pytest.raises(B.DEError) as ei:   # nu out of range
        B.de_setup(2, (32, 16), 1.0, p.fixed, p.density, 1.0, 1e-9, 3.0, 0.5, (16, 8))
    assert ei.value.status == B.DE_EINVAL
    with pytest.raises(B.DEError) as ei:   # no Dirichlet dof
        B.de_setup(2, (32, 16), 1.0, np.zeros_like(p.fixed), p.density, 1.0, 1e-9, 3.0, 0.3, (16, 8))
    assert ei.value.status == B.DE_EINVAL
    rho = p.density.copy()
    rho[3] = 0.0                            # rho <= 0
    with pytest.raises(B.DEError) as ei:
        B.de_setup(2, (32, 16), 1.0, p.fixed, rho, 1.0, 1e-9, 3.0, 0.3, (16, 8))
    assert ei.value.status == B.DE_EINVAL
