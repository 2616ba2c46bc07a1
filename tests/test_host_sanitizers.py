"""The host coders under AddressSanitizer + UndefinedBehaviorSanitizer (decoders fed thousands
of truncated / bit-flipped streams) and ThreadSanitizer (8 threads coding concurrently with
shared prepared tables), SURVEY.md §5 -- -m "not gpu".  Built from the product sources with
g++ (tests/host_sanitize.cpp)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRCS = [os.path.join(ROOT, "paper_2208_01641_b200", "csrc", f) for f in ("host_coder.cpp", "host_rans64.cpp")]


def _build(tmp_path, name, flags):
    exe = str(tmp_path / name)
    cmd = ["g++", "-O1", "-g", "-std=c++17", "-pthread", *flags, f"-I{os.path.join(ROOT, 'include')}",
           os.path.join(ROOT, "tests", "host_sanitize.cpp"), *SRCS, "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        pytest.skip(f"sanitizer build unavailable: {r.stderr[-300:]}")
    return exe


@pytest.mark.skipif(shutil.which("g++") is None, reason="no g++")
def test_decoders_under_asan_ubsan(tmp_path):
    exe = _build(tmp_path, "san_asan", ["-fsanitize=address,undefined", "-fno-sanitize-recover=all"])
    r = subprocess.run([exe, "fuzz"], capture_output=True, text=True, timeout=300,
                       env={**os.environ, "LIC_NO_AVX512": "0"})
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]


@pytest.mark.skipif(shutil.which("g++") is None, reason="no g++")
def test_scalar_decoders_under_asan_ubsan(tmp_path):
    exe = _build(tmp_path, "san_asan_scalar", ["-fsanitize=address,undefined", "-fno-sanitize-recover=all"])
    r = subprocess.run([exe, "fuzz"], capture_output=True, text=True, timeout=300,
                       env={**os.environ, "LIC_NO_AVX512": "1"})
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]


@pytest.mark.skipif(shutil.which("g++") is None, reason="no g++")
def test_concurrent_coders_under_tsan(tmp_path):
    exe = _build(tmp_path, "san_tsan", ["-fsanitize=thread"])
    r = subprocess.run([exe, "threads"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "WARNING: ThreadSanitizer" not in r.stderr, r.stdout[-2000:] + r.stderr[-4000:]
