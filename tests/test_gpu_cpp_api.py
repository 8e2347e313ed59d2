"""The reference-side C++ API (include/pswa/pipeline.h) drives the device
path: encode_frame -> decode_frame_wavefront over a synthetic GOP,
bit-exact (examples/decode_gop.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "paper_2605_20977_b200", "build", "decode_gop")


@pytest.mark.gpu
@pytest.mark.parametrize("args", [["16", "16", "0", "5"], ["20", "24", "1", "2"]])
def test_cpp_pipeline_roundtrip(args):
    r = subprocess.run([EXE] + args, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count(" ok:") == int(args[3])


def test_cpp_example_built():
    assert os.path.exists(EXE), "build() must produce the C++ example"
