"""The C++ façade (include/slimsell_b200/*.hpp) through its own test binary:
compiled here (CPU), run against the device on a B200 (gpu)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2010_09913_b200")
ORACLE = os.path.join(ROOT, "oracle")


@pytest.fixture(scope="module")
def facade_binary(tmp_path_factory):
    from oracle import build as build_oracle
    from paper_2010_09913_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        _lib.build()
    if not os.path.exists(os.path.join(ORACLE, "liboracle.so")):
        build_oracle(ref=False)
    exe = tmp_path_factory.mktemp("cpp") / "test_facade"
    cmd = ["g++", "-std=c++20", "-O1", "-Wall", "-I", os.path.join(ROOT, "include"), "-I", ORACLE,
           os.path.join(ROOT, "tests", "cpp", "test_facade.cpp"), "-o", str(exe),
           "-L", PKG, "-lslimsell_b200", "-L", ORACLE, "-loracle",
           f"-Wl,-rpath,{PKG}", f"-Wl,-rpath,{ORACLE}"]
    out = subprocess.run(cmd, capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    return str(exe)


def test_facade_compiles_and_links(facade_binary):
    assert os.path.exists(facade_binary)


@pytest.mark.gpu
def test_facade_parity_on_device(facade_binary):
    out = subprocess.run([facade_binary], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert " 0 failed" in out.stdout


ALONGSIDE = os.path.join(ORACLE, "_ref", "test_alongside")


def test_alongside_reference_compiles_and_links():
    """The façade and the reference's own headers in ONE translation unit
    (SLIMSELL_B200_ALONGSIDE_REFERENCE), linked with the reference library;
    built where /root/reference exists, run on the B200 below."""
    from oracle import build as build_oracle
    from oracle.cpu import REF_DIR
    from paper_2010_09913_b200 import _lib
    if not os.path.isdir(REF_DIR):
        pytest.skip("needs the reference sources (this container)")
    if not os.path.exists(_lib.LIB_PATH):
        _lib.build()
    build_oracle(ref=True, alongside=True)
    out = subprocess.run([ALONGSIDE], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr  # no device here: prints and exits 0


@pytest.mark.gpu
def test_alongside_reference_on_device():
    """Reference-built host layouts, the reference's CsrView / SemiringSpec and
    an in-place corrupted layout through the façade: equal to the reference's
    own calls on the same objects."""
    if not os.path.exists(ALONGSIDE):
        pytest.skip("oracle/_ref/test_alongside not built (build() builds it where the reference exists)")
    out = subprocess.run([ALONGSIDE], capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stdout + out.stderr
    assert " 0 failed" in out.stdout, out.stdout
