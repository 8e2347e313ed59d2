"""Host-side drop-in headers, no GPU: validate_schedule (pswa/wavefront.h,
reference proj/include/pswa/wavefront.h:54-66) and
parallel_for (pswa/threading.h, reference threading.h:24-31).
The C++ checks (broken predicates, thread-pool semantics) run as
paper_2605_20977_b200/build/test_host_api; the C-ABI validate_schedule is
compared with the oracle's restatement on a grid sweep."""
import ctypes as C
import os
import subprocess

import pytest

from oracle_api import oracle
from paper_2605_20977_b200 import lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_2605_20977_b200", "build", "test_host_api")


def test_cpp_host_api_checks():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.strip().startswith("ok")


def product_validate(h, w, s, wh, ww, n):
    ok, steps = C.c_int(), C.c_int()
    msg = C.create_string_buffer(512)
    L = lib()
    L.pswa_validate_schedule.argtypes = [C.c_int] * 6 + [C.c_void_p, C.c_void_p, C.c_char_p, C.c_size_t]
    assert L.pswa_validate_schedule(h, w, s, wh, ww, n, C.byref(ok), C.byref(steps), msg, 512) == 0
    return ok.value, steps.value, msg.value.decode()


@pytest.mark.parametrize("h,w", [(1, 1), (4, 4), (7, 5), (16, 16), (8, 33), (64, 64)])
@pytest.mark.parametrize("s", [1, 2, 3, 4, 8])
def test_validate_schedule_matches_oracle(h, w, s):
    for n in (1, 4):
        ok, steps, _ = product_validate(h, w, s, 7, 7, n)
        so = C.c_int()
        ok_o = oracle().oracle_validate_schedule(h, w, s, 7, 7, n, C.byref(so))
        assert (ok, steps) == (ok_o, so.value) == (1, s * n)


def test_validate_schedule_rejects_bad_parameters():
    ok, _, msg = product_validate(8, 8, 4, 6, 7, 4)  # even window extent
    assert ok == 0 and "precondition" in msg
    ok, _, msg = product_validate(8, 8, 0, 7, 7, 4)
    assert ok == 0 and "precondition" in msg
