"""Sequence container host logic (FORMAT.md §1) on the CPU:
header fields, whole-frame framing of truncated streams, bad headers."""
import os
import struct

import numpy as np
import pytest

from paper_2605_20977_b200 import PswaError
from paper_2605_20977_b200.codec import container_info

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "seq_desk_8x8.pswa")


def _container(frames):
    hdr = b"PSWA" + struct.pack("<HH7IQQIII", 3, 64, 128, 96, len(frames), 2, 1, 4, 4,
                                0x1234, 0x5678, 1, 1, 0)
    body = b"".join(struct.pack("<I", len(h)) + h + struct.pack("<I", len(m)) + m
                    for h, m in frames)
    return hdr + body


def test_header_fields_and_framing():
    c = _container([(b"a" * 10, b"b" * 20), (b"c" * 3, b"d" * 7), (b"e", b"f" * 5)])
    info = container_info(c)
    assert info["version"] == 3 and info["w_px"] == 128 and info["h_px"] == 96
    assert info["frames"] == 3 and info["gop"] == 2 and info["rate"] == 1
    assert info["s"] == 4 and info["N"] == 4 and info["prior"] == 1
    assert info["frames_present"] == 3
    # truncation inside frame 2 (any byte short) keeps the 2 whole frames
    for cut in (1, 3, 6):
        assert container_info(c[:-cut])["frames_present"] == 2
    assert container_info(c[:64])["frames_present"] == 0


def test_bad_headers_rejected():
    c = _container([(b"x", b"y")])
    with pytest.raises(PswaError):
        container_info(b"XSWA" + c[4:])
    with pytest.raises(PswaError):
        container_info(c[:4] + struct.pack("<H", 4) + c[6:])  # unknown version
    with pytest.raises(PswaError):
        container_info(c[:40])  # shorter than the header


@pytest.mark.skipif(not os.path.exists(GOLDEN), reason="golden container not generated yet")
def test_golden_container_header():
    info = container_info(open(GOLDEN, "rb").read())
    assert info["frames"] == info["frames_present"] == 3
    assert info["gop"] == 2 and info["rate"] == 1 and info["w_px"] == 128 and info["h_px"] == 128


@pytest.mark.parametrize("old", [1, 2])
def test_other_numerics_revision_refused(old):
    """Versions 1 and 2 were coded under earlier numerics (round-1 SiLU /
    softplus; the unsplit down projection): refused, never decoded to wrong
    latents."""
    c = _container([(b"a" * 10, b"b" * 20)])
    with pytest.raises(PswaError) as e:
        container_info(c[:4] + struct.pack("<H", old) + c[6:])
    assert "version" in str(e.value)
