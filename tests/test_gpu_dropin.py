"""GPU: the reference's OWN doctest suites (tests/test_pir.cpp, test_cuckoo.cpp,
test_server.cpp from /root/reference/proj, compiled as they lie by
`make -C oracle dropin`) linked against the B200 drop-in translation units
paper_2001_08250_b200/cpp/{pir,cuckoo}_b200.cpp in place of src/pir.cpp and
src/cuckoo.cpp. Every PIR answer, mask and cuckoo insert in those suites runs on
the GPU through include/xpir.h.

The same suites are also linked against the unmodified reference TUs
(test_*_ref). The drop-in must reproduce the reference run exactly: same cases,
same checks, same failures. (The unmodified reference fails one case of its own
test_server.cpp — "window freezes appear on the rotation cadence", five checks
on freeze indices — independently of the PIR/cuckoo path; the drop-in build
must fail exactly those checks and nothing else.)"""
import os
import re
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DROPIN = os.path.join(ROOT, "oracle", "_ref", "dropin")


def run(exe):
    out = subprocess.run([exe], capture_output=True, text=True, timeout=1200)
    fails = sorted(set(re.findall(r"(\S+:\d+: CHECK FAILED: .*)", out.stderr)))
    cases = sorted(set(re.findall(r"TEST CASE FAILED: (.*)", out.stderr)))
    summary = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed \| checks: (\d+) \| (\d+) failed",
                        out.stdout)
    return out, fails, cases, summary


@pytest.mark.parametrize("suite", ["test_pir", "test_cuckoo", "test_server"])
def test_reference_suite_against_dropin(suite, cuda):
    exe_b200 = os.path.join(DROPIN, suite + "_b200")
    exe_ref = os.path.join(DROPIN, suite + "_ref")
    if not os.path.exists(exe_b200) or not os.path.exists(exe_ref):
        pytest.skip("drop-in suites not built (needs /root/reference at build time)")
    out_b, fails_b, cases_b, sum_b = run(exe_b200)
    out_r, fails_r, cases_r, sum_r = run(exe_ref)
    print(out_b.stdout[-500:], out_b.stderr[-3000:])
    assert out_b.returncode in (0, 1), f"drop-in suite crashed: rc={out_b.returncode}\n{out_b.stderr[-3000:]}"
    assert sum_b is not None and sum_r is not None
    assert fails_b == fails_r and cases_b == cases_r
    assert sum_b.group(1) == sum_r.group(1) and sum_b.group(3) == sum_r.group(3)
    assert sum_b.group(4) == sum_r.group(4)  # same number of checks executed
    assert out_b.returncode == out_r.returncode
    if suite != "test_server":
        assert out_b.returncode == 0 and sum_b.group(3) == "0"


def test_concurrent_reads_through_dropin(cuda):
    """64 threads x 12 pir::answer + mask_answer calls on one Snapshot through the
    drop-in TU (the read batcher coalesces them); host-XOR checker."""
    exe = os.path.join(DROPIN, "dropin_mt_b200")
    if not os.path.exists(exe):
        pytest.skip("drop-in binaries not built (needs /root/reference at build time)")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(out.stdout, out.stderr[-2000:])
    assert out.returncode == 0 and "0 mismatches" in out.stdout
