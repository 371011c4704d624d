"""GPU: the reference's OWN doctest suites (tests/test_pir.cpp, test_cuckoo.cpp,
test_server.cpp from /root/reference/proj, compiled as they lie by
`make -C oracle dropin`) linked against the B200 drop-in translation units
paper_2001_08250_b200/cpp/{pir,cuckoo}_b200.cpp in place of src/pir.cpp and
src/cuckoo.cpp. Every PIR answer, mask and cuckoo insert in those suites runs on
the GPU through include/xpir.h."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DROPIN = os.path.join(ROOT, "oracle", "_ref", "dropin")


@pytest.mark.parametrize("suite", ["test_pir_b200", "test_cuckoo_b200", "test_server_b200"])
def test_reference_suite_against_dropin(suite, cuda):
    exe = os.path.join(DROPIN, suite)
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built (needs /root/reference at build time)")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=1200)
    print(out.stdout[-2000:])
    print(out.stderr[-4000:])
    assert out.returncode == 0, out.stderr[-4000:]
    assert "0 failed" in out.stdout
