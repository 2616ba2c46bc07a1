"""The C-ABI library builds, loads and exports every symbol include/lic.h declares
(-m "not gpu": no compute calls that need a GPU)."""
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "lic.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lic_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2208_01641_b200 import build
    build.build()
    from paper_2208_01641_b200 import lic
    L = lic.lib()
    names = declared_symbols()
    assert len(names) >= 20
    for n in names:
        assert hasattr(L, n), n
    assert "sm_100a" in lic.version()


def test_cubin_is_sm100a_with_tcgen05():
    """The engine kernel is real sm_100a tcgen05/TMA code (SASS UTCHMMA / UTMALDG)."""
    import subprocess
    from paper_2208_01641_b200 import build
    lib = build.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "UTCHMMA" in out or "UTCQMMA" in out
    assert "UTMALDG" in out
    assert "LDTM" in out


def test_open_without_gpu_fails_loudly():
    """No GPU (this container): lic_open must refuse (LIC_ECUDA), never fall back."""
    import torch
    if torch.cuda.is_available():
        return
    from lic_synth import ModelSpec, generate_weights, write_licw
    from paper_2208_01641_b200 import lic
    spec = ModelSpec(kind=0, N=128, M=192)
    blob = write_licw(spec, generate_weights(spec, 0))
    try:
        lic.Codec(blob, 64, 64)
    except lic.LicError as e:
        assert e.status == lic.LIC_ECUDA
    else:
        raise AssertionError("lic_open succeeded without a GPU")


def test_invalid_weights_rejected_before_device():
    """SPEC.md:102 (beta > 0, gamma >= 0 validated at load) and a malformed container are
    rejected by lic_open's parser, before any device work."""
    import numpy as np
    from lic_synth import ModelSpec, generate_weights, write_licw
    from paper_2208_01641_b200 import lic
    spec = ModelSpec(kind=1, N=128, M=192)
    w = generate_weights(spec, 0)
    w["ga2.beta"] = w["ga2.beta"].copy()
    w["ga2.beta"][3] = 0.0
    try:
        lic.Codec(write_licw(spec, w), 128, 128)
    except lic.LicError as e:
        assert e.status == lic.LIC_EINVAL
    else:
        raise AssertionError("beta = 0 accepted")
    w = generate_weights(spec, 0)
    w["gs1.gamma"] = w["gs1.gamma"].copy()
    w["gs1.gamma"][0, 5] = -0.01
    try:
        lic.Codec(write_licw(spec, w), 128, 128)
    except lic.LicError as e:
        assert e.status == lic.LIC_EINVAL
    blob = write_licw(spec, generate_weights(spec, 0))
    for bad in (blob[:-4], b"LICX" + blob[4:], blob + b"\0"):
        try:
            lic.Codec(bad, 128, 128)
        except lic.LicError as e:
            assert e.status == lic.LIC_EDIGEST
        else:
            raise AssertionError("malformed container accepted")
