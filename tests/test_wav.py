"""wav.py against hand-built files, mirroring the reference's test_wav.cpp case by case (CPU only)."""
import struct

import numpy as np
import pytest

from paper_2212_05271_b200.gss import IoError, ParseError, wav
from paper_2212_05271_b200.gss.stft import RealSignal
from .refrng import Rng


def write_pcm(path, bits, channels, rate, interleaved):
    """Minimal independent writer (test_wav.cpp:27-50): the reader is tested against bytes it did not write."""
    nbytes = bits // 8
    data = b"".join(struct.pack("<i", v)[:nbytes] for v in interleaved)
    with open(path, "wb") as f:
        f.write(b"RIFF" + struct.pack("<I", 36 + len(data)) + b"WAVE" + b"fmt " + struct.pack("<I", 16))
        f.write(struct.pack("<HHIIHH", 1, channels, rate, rate * channels * nbytes, channels * nbytes, bits))
        f.write(b"data" + struct.pack("<I", len(data)) + data)


def test_float32_round_trip_is_bit_exact(tmp_path):  # test_wav.cpp:58-85
    rng = Rng(7)
    x = np.array([[np.float32(rng.uniform() * 2 - 1) for _ in range(997)] for _ in range(3)], dtype=np.float32)
    path = str(tmp_path / "roundtrip.wav")
    wav.write(path, RealSignal(x, 16000))
    wi = wav.info(path)
    assert (wi.channels, wi.sample_rate, wi.format, wi.bits_per_sample, wi.num_frames) == (3, 16000, 3, 32, 997)
    back = wav.read(path)
    assert back.num_channels() == 3 and back.num_samples() == 997
    assert back.channels.tobytes() == x.tobytes()


def test_windowed_read(tmp_path):  # test_wav.cpp:87-106
    path = str(tmp_path / "ramp.wav")
    wav.write(path, RealSignal(np.arange(100, dtype=np.float32).reshape(1, -1), 8000))
    win = wav.read(path, 10, 5)
    assert win.num_samples() == 5 and np.array_equal(win.channels[0], np.arange(10, 15, dtype=np.float32))
    assert wav.read(path, 95).num_samples() == 5  # max_frames < 0 reads to the end
    with pytest.raises(IoError):
        wav.read(path, 200, 1)


def test_pcm16_scales_by_32768(tmp_path):  # test_wav.cpp:112-123
    path = str(tmp_path / "pcm16.wav")
    write_pcm(path, 16, 2, 16000, [16384, -32768, 0, 32767])
    s = wav.read(path)
    assert s.num_channels() == 2 and s.num_samples() == 2
    assert s.channels[0][0] == 0.5 and s.channels[1][0] == -1.0 and s.channels[0][1] == 0.0
    assert s.channels[1][1] == np.float32(32767.0) / np.float32(32768.0)


def test_pcm24_sign_extension(tmp_path):  # test_wav.cpp:125-133
    path = str(tmp_path / "pcm24.wav")
    write_pcm(path, 24, 1, 16000, [0x400000, -0x800000, -1])
    s = wav.read(path)
    assert s.num_samples() == 3
    assert s.channels[0][0] == 0.5 and s.channels[0][1] == -1.0
    assert s.channels[0][2] == np.float32(-1.0) / np.float32(8388608.0)


def test_unsupported_and_malformed_files(tmp_path):  # test_wav.cpp:139-161
    p8 = str(tmp_path / "pcm8.wav")
    write_pcm(p8, 8, 1, 16000, [1, 2, 3])
    with pytest.raises(ParseError):
        wav.info(p8)
    garbage = tmp_path / "garbage.wav"
    garbage.write_bytes(b"not a riff file")
    with pytest.raises(ParseError):
        wav.info(str(garbage))
    truncated = tmp_path / "truncated.wav"
    truncated.write_bytes(b"RIFF\x04\x00\x00\x00WAVE")  # no fmt / data chunks
    with pytest.raises(ParseError):
        wav.info(str(truncated))
    with pytest.raises(IoError):
        wav.info(str(tmp_path / "does_not_exist.wav"))


def test_reader_skips_unknown_and_odd_sized_chunks(tmp_path):  # test_wav.cpp:163-190
    path = tmp_path / "chunky.wav"
    body = (b"WAVE" + b"junk" + struct.pack("<I", 3) + b"abc\0" + b"fmt " + struct.pack("<I", 16)
            + struct.pack("<HHIIHH", 1, 1, 16000, 32000, 2, 16) + b"data" + struct.pack("<I", 4)
            + struct.pack("<HH", 0x4000, 0xC000))
    path.write_bytes(b"RIFF" + struct.pack("<I", len(body)) + body)
    s = wav.read(str(path))
    assert s.num_samples() == 2 and s.channels[0][0] == 0.5 and s.channels[0][1] == -0.5


def test_extensible_format_uses_the_subformat_tag(tmp_path):  # wav.hpp:77-80
    path = tmp_path / "ext.wav"
    fmt = struct.pack("<HHIIHH", 0xFFFE, 1, 16000, 64000, 4, 32) + struct.pack("<HHI", 22, 32, 4)
    fmt += struct.pack("<H", 3) + b"\x00" * 14  # sub-format GUID leads with the tag (3 = IEEE float)
    data = np.array([0.25, -0.75], dtype="<f4").tobytes()
    body = b"WAVE" + b"fmt " + struct.pack("<I", len(fmt)) + fmt + b"data" + struct.pack("<I", len(data)) + data
    path.write_bytes(b"RIFF" + struct.pack("<I", len(body)) + body)
    wi = wav.info(str(path))
    assert wi.format == 3 and wi.num_frames == 2
    assert np.array_equal(wav.read(str(path)).channels[0], np.array([0.25, -0.75], dtype=np.float32))
