"""wav.hpp: RIFF/WAVE reader (PCM16, PCM24, IEEE float32, WAVE_FORMAT_EXTENSIBLE, odd-sized chunks) and the
float32 writer the pipeline uses for its outputs (wav.hpp:50-181). Host-side file format, no device work."""
from __future__ import annotations

import os
import struct
from dataclasses import dataclass

import numpy as np

from .common import IoError, ParseError, ShapeError
from .stft import RealSignal


@dataclass
class WavInfo:  # wav.hpp:14-22
    channels: int = 0
    sample_rate: int = 0
    bits_per_sample: int = 0
    format: int = 0          # 1 = PCM, 3 = IEEE float
    num_frames: int = 0
    data_offset: int = 0
    data_bytes: int = 0


def info(path: str) -> WavInfo:  # wav.hpp:50-104
    try:
        f = open(path, "rb")
    except OSError:
        raise IoError("cannot open wav file: " + path)
    with f:
        header = f.read(12)
        if len(header) < 12 or header[:4] != b"RIFF" or header[8:12] != b"WAVE":
            raise ParseError("not a RIFF/WAVE file: " + path)
        wi = WavInfo()
        have_fmt = False
        while True:
            chunk = f.read(8)
            if len(chunk) < 8:
                break
            size = struct.unpack("<I", chunk[4:8])[0]
            body = f.tell()
            if chunk[:4] == b"fmt ":
                fmt = f.read(size)
                if size < 16 or len(fmt) < size:
                    raise ParseError("truncated fmt chunk: " + path)
                wi.format, wi.channels, wi.sample_rate = struct.unpack("<HHI", fmt[:8])
                wi.bits_per_sample = struct.unpack("<H", fmt[14:16])[0]
                if wi.format == 0xFFFE:  # extensible: the sub-format GUID leads with the tag
                    if size < 40:
                        raise ParseError("truncated extensible fmt: " + path)
                    wi.format = struct.unpack("<H", fmt[24:26])[0]
                have_fmt = True
            elif chunk[:4] == b"data":
                wi.data_offset = body
                wi.data_bytes = size
                break
            else:
                f.seek(body + size + (size & 1))  # chunks are padded to even sizes
        if not have_fmt or wi.data_offset == 0:
            raise ParseError("wav missing fmt or data chunk: " + path)
        if wi.channels < 1 or wi.bits_per_sample < 1:
            raise ParseError("wav has invalid fmt fields: " + path)
        supported = (wi.format == 1 and wi.bits_per_sample in (16, 24)) or (wi.format == 3 and wi.bits_per_sample == 32)
        if not supported:
            raise ParseError("unsupported wav encoding (format %d, %d bit): %s" % (wi.format, wi.bits_per_sample, path))
        block = wi.channels * wi.bits_per_sample // 8
        wi.num_frames = wi.data_bytes // block
        return wi


def read(path: str, start_frame: int = 0, max_frames: int = -1) -> RealSignal:  # wav.hpp:108-151
    """[start_frame, start_frame + max_frames) as float32 channels; max_frames < 0 = the rest of the file."""
    wi = info(path)
    if start_frame < 0 or start_frame > wi.num_frames:
        raise IoError("wav read window starts at %d of %d frames: %s" % (start_frame, wi.num_frames, path))
    count = wi.num_frames - start_frame
    if max_frames >= 0:
        count = min(count, max_frames)
    bps = wi.bits_per_sample // 8
    block = wi.channels * bps
    try:
        with open(path, "rb") as f:
            f.seek(wi.data_offset + start_frame * block)
            raw = f.read(count * block)
    except OSError:
        raise IoError("cannot open wav file: " + path)
    if len(raw) < count * block:
        raise IoError("short read from wav data: " + path)
    if wi.format == 3:
        x = np.frombuffer(raw, dtype="<f4").reshape(count, wi.channels)
    elif wi.bits_per_sample == 16:
        x = np.frombuffer(raw, dtype="<i2").reshape(count, wi.channels).astype(np.float32) / np.float32(32768.0)
    else:  # 24-bit PCM, sign-extended
        b = np.frombuffer(raw, dtype=np.uint8).reshape(count, wi.channels, 3).astype(np.int32)
        s = b[..., 0] | (b[..., 1] << 8) | (b[..., 2] << 16)
        s = np.where(s & 0x800000, s - (1 << 24), s)
        x = s.astype(np.float32) / np.float32(8388608.0)
    return RealSignal(np.ascontiguousarray(x.T, dtype=np.float32), wi.sample_rate)


def write(path: str, signal: RealSignal) -> None:  # wav.hpp:154-181
    """IEEE float32 WAV, channels interleaved; truncates an existing file."""
    channels = signal.num_channels()
    frames = signal.num_samples()
    if channels < 1:
        raise ShapeError("wav.write: no channels")
    data = np.ascontiguousarray(np.asarray(signal.channels, dtype=np.float32).T).astype("<f4", copy=False)
    data_bytes = (frames * channels * 4) & 0xFFFFFFFF
    sr = int(signal.sample_rate) & 0xFFFFFFFF
    header = (b"RIFF" + struct.pack("<I", (36 + data_bytes) & 0xFFFFFFFF) + b"WAVE" + b"fmt "
              + struct.pack("<IHHIIHH", 16, 3, channels, sr, (sr * channels * 4) & 0xFFFFFFFF, channels * 4, 32)
              + b"data" + struct.pack("<I", data_bytes))
    try:
        with open(path, "wb") as f:
            f.write(header)
            f.write(data.tobytes())
    except OSError as e:
        if not os.path.isdir(os.path.dirname(path) or "."):
            raise IoError("cannot create wav file: " + path)
        raise IoError("failed writing wav data: %s (%s)" % (path, e))
