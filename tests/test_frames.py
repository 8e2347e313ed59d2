"""Frames (SPEC.md:499-548 toy transform, :663-670 PPM). CPU: PPM round trip,
P3 / bad headers rejected, replicate-edge padding. GPU (marked): the device
DCT against a float64 numpy restatement, constant-gray -> DC channels only,
orthonormal round trip and Parseval, and an end-to-end sequence
(frames -> container -> frames) with the LRP transformer."""
import os

import numpy as np
import pytest

from paper_2605_20977_b200 import PswaError
from paper_2605_20977_b200 import frames as fr

ZIG = [0, 1, 8, 16, 9, 2, 3, 10, 17, 24, 32, 25, 18, 11, 4, 5, 12, 19, 26, 33, 40, 48, 41, 34, 27,
       20, 13, 6, 7, 14, 21, 28, 35, 42, 49, 56, 57, 50, 43, 36, 29, 22, 15, 23, 30, 37, 44, 51,
       58, 59, 52, 45, 38, 31, 39, 46, 53, 60, 61, 54, 47, 55, 62, 63]
Q = [8.0, 5.0, 3.0, 2.0]


def _dct_mat():
    k, n = np.meshgrid(np.arange(8), np.arange(8), indexing="ij")
    m = np.sqrt(2 / 8) * np.cos((2 * n + 1) * k * np.pi / 16)
    m[0] /= np.sqrt(2)
    return m  # [k][n]


def _analysis_ref(rgb, rate):
    D = _dct_mat()
    h, w = rgb.shape[0] // 8, rgb.shape[1] // 8
    x = rgb.astype(np.float64) - 128.0
    y = np.zeros((192, h, w))
    for py in range(h):
        for px in range(w):
            for c in range(3):
                blk = D @ x[py * 8:py * 8 + 8, px * 8:px * 8 + 8, c] @ D.T
                for z in range(64):
                    y[z * 3 + c, py, px] = blk[ZIG[z] // 8, ZIG[z] % 8]
    return y / Q[rate]


def _test_image(h=32, w=48, seed=0):
    yy, xx = np.mgrid[0:h, 0:w]
    rng = np.random.default_rng(seed)
    img = np.stack([(xx * 5) % 256, (yy * 7) % 256, ((xx + yy) * 3) % 256], -1).astype(np.float64)
    img[8:20, 10:30] = [200, 40, 90]
    img += rng.normal(0, 6, img.shape)
    return np.clip(np.rint(img), 0, 255).astype(np.uint8)


def test_ppm_roundtrip_and_rejections(tmp_path):
    img = _test_image(13, 17)
    p = str(tmp_path / "a.ppm")
    fr.write_ppm(p, img)
    assert np.array_equal(fr.read_ppm(p), img)
    p3 = tmp_path / "b.ppm"
    p3.write_bytes(b"P3\n2 2\n255\n0 0 0 0 0 0 0 0 0 0 0 0\n")
    with pytest.raises(PswaError):
        fr.read_ppm(str(p3))
    bad = tmp_path / "c.ppm"
    bad.write_bytes(b"P6\n2 2\n65535\n" + bytes(24))
    with pytest.raises(PswaError):
        fr.read_ppm(str(bad))
    trunc = tmp_path / "d.ppm"
    trunc.write_bytes(b"P6\n# comment\n4 4\n255\n" + bytes(10))
    with pytest.raises(PswaError):
        fr.read_ppm(str(trunc))


def test_pad8_replicates_edges():
    img = _test_image(13, 17)
    p = fr.pad8(img)
    assert p.shape == (16, 24, 3)
    assert np.array_equal(p[:13, :17], img)
    assert np.array_equal(p[13:, :17], np.repeat(img[12:13], 3, 0))
    assert np.array_equal(p[:13, 17:], np.repeat(img[:, 16:17], 7, 1))


@pytest.mark.gpu
def test_toy_transform_on_device():
    img = _test_image()
    for rate in range(4):
        y = fr.analysis(img, rate)
        assert np.abs(y - _analysis_ref(img, rate)).max() < 2e-3
    gray = np.full((16, 16, 3), 77, np.uint8)
    yg = fr.analysis(gray, 0)
    assert np.abs(yg[3:]).max() < 1e-4 and np.abs(yg[:3]).min() > 1.0  # DC channels only
    y = fr.analysis(img, 3)
    assert np.array_equal(fr.synthesis(y, 3), img)  # no quantisation: exact after rounding
    x = img.astype(np.float64) - 128.0
    assert abs((y.astype(np.float64) ** 2).sum() * Q[3] ** 2 / (x ** 2).sum() - 1) < 1e-2  # Parseval
    # coarser quantisation, lower PSNR
    def psnr(a, b):
        return 10 * np.log10(255 ** 2 / np.mean((a.astype(float) - b) ** 2))
    p = [psnr(fr.synthesis(np.rint(fr.analysis(img, r)), r), img) for r in (0, 3)]
    assert p[1] > p[0]


@pytest.mark.gpu
def test_frames_end_to_end_with_lrp(tmp_path):
    from oracle_api import gen_weights, preset
    from paper_2605_20977_b200.codec import GpuCodec, cfg_from_dict
    imgs = [_test_image(64, 64, seed=s) for s in range(3)]
    c = preset(False, 8, 8, lanes=8, hyper_lanes=4, lrp_blocks=1)
    cfg = cfg_from_dict(c)
    blob = gen_weights(c, 1)
    cont = fr.encode_frames(GpuCodec(cfg, blob), imgs, gop=2, rate=2)
    rgb, ys = fr.decode_frames(GpuCodec(cfg, blob), cont)
    for img, y, out in zip(imgs, ys, rgb):
        assert np.array_equal(y, fr.quantize(fr.analysis(img, 2)))  # latents bit-exact
        assert out.shape == img.shape
        # reconstruction error bounded by quantisation (+ |eps| < 0.5 per latent)
        assert np.mean(np.abs(out.astype(float) - img)) < 6.0
    fr.write_ppm(str(tmp_path / "rec.ppm"), rgb[0])
