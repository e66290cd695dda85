"""The kvpack v1 container around the device-packed sections.

Byte-identical to the reference writer (kvpack.py:7-37,126-177): 128-byte
little-endian header, section table of 5 x (offset u64, length u64), the
sections in order (scales, indices, radii, flags, payloads), CRC-32 trailer.
The section bit streams are produced by the encode kernel in HBM already in
their serialized form (LSB-first, byte-aligned starts), so to_bytes is a
device->host copy plus the header and checksum; from_bytes validates like
the reference reader (kvpack.py:194-306) and uploads the sections, deriving
the per-token coded offsets and checking every index on the GPU.
"""

from __future__ import annotations

import ctypes
import struct

import numpy as np

from . import _native as nat
from .codebook import ROLE_TAGS
from .codec import CHUNK_DIM, CodecConfig, QuantizedTensor, TensorShape, _words
from .errors import CorruptData, InvalidArgument, UnsupportedVersion

MAGIC = b"HQMQ"
VERSION = 1
HEADER_BYTES = 128
_HEADER_FMT = "<4sHHIIIIIBBHQII"
_SECTION_COUNT = 5
_FLAG_OUTLIER = 1
_FLAG_PER_HEAD = 2


def _multiplier_to_fixed(multiplier) -> int:
    if multiplier is None:
        return 0
    fixed = int(round(multiplier * 65536.0))
    if not 0 < fixed <= 0xFFFFFFFF:
        raise InvalidArgument(f"outlier multiplier {multiplier} not representable")
    return fixed


def expected_file_size(packed: QuantizedTensor) -> int:
    """kvpack.py:99-112."""
    s, c = packed.shape, packed.config
    n = s.n_chunks
    n_coded = packed.n_coded
    size = HEADER_BYTES + 2 * s.batch * s.heads * s.tokens
    size += (n_coded * c.index_bits + 7) // 8
    size += (n_coded * c.radius_bits + 7) // 8
    if c.outlier_multiplier is not None:
        size += (n + 7) // 8
    size += 8 * packed.n_payload
    return size + 4


def _header(packed: QuantizedTensor, lengths) -> bytes:
    """128-byte header + section table (kvpack.py:126-175)."""
    s, c = packed.shape, packed.config
    flags = (_FLAG_OUTLIER if c.outlier_multiplier is not None else 0) | (
        _FLAG_PER_HEAD if c.median_pooling == "per_head" else 0)
    header = struct.pack(_HEADER_FMT, MAGIC, VERSION, flags, s.batch, s.heads, s.tokens,
                         s.head_dim, c.codebook_size, c.radius_bits, ROLE_TAGS[packed.role],
                         packed.head_base, c.seed, _multiplier_to_fixed(c.outlier_multiplier),
                         packed.layer)
    table = bytearray()
    off = HEADER_BYTES
    for n in lengths:
        table += struct.pack("<QQ", off, n)
        off += n
    return header + bytes(table)


def device_crc32(buf, n: int, out) -> None:
    """zlib.crc32 of the first n bytes of a uint8 CUDA tensor, written
    little-endian into the 4-byte uint8 CUDA tensor `out` (hqmq_crc32)."""
    import torch

    L = nat.lib()
    ws = torch.empty(int(L.hqmq_crc32_workspace_bytes(n)), dtype=torch.uint8, device=buf.device)
    nat.launch(buf.device, "hqmq_crc32", L.hqmq_crc32, buf.data_ptr(), n, out.data_ptr(),
               ws.data_ptr(), ws.numel())
    buf._crc_ws = ws  # keep the workspace alive until the stream has used it


def to_device_image(packed: QuantizedTensor):
    """The whole kvpack file assembled in HBM (header, section table, the five
    sections copied device-to-device, CRC-32 computed on the GPU): a uint8
    CUDA tensor whose bytes equal the reference's to_bytes (kvpack.py:126-177)."""
    import torch

    s, c = packed.shape, packed.config
    if packed.role not in ROLE_TAGS:
        raise InvalidArgument(f"role must be one of {sorted(ROLE_TAGS)}")
    if not 0 <= packed.head_base + s.heads <= 0xFFFF:
        raise InvalidArgument("head_base + heads must fit in 16 bits")
    n_coded = packed.n_coded  # synchronises the encode and raises its errors
    dev = packed.device
    as_u8 = lambda t: t.contiguous().view(-1).view(torch.uint8)  # noqa: E731
    secs = [as_u8(packed.scales),
            as_u8(packed.index_words)[: (n_coded * c.index_bits + 7) // 8],
            as_u8(packed.radius_words)[: (n_coded * c.radius_bits + 7) // 8],
            as_u8(packed.flag_words)[: (s.n_chunks + 7) // 8]
            if c.outlier_multiplier is not None else None,
            as_u8(packed.payloads) if packed.n_payload else None]
    lengths = [0 if t is None else t.numel() for t in secs]
    head = _header(packed, lengths)
    total = len(head) + sum(lengths)
    img = torch.empty(total + 4, dtype=torch.uint8, device=dev)
    img[: len(head)].copy_(torch.frombuffer(bytearray(head), dtype=torch.uint8), non_blocking=False)
    off = len(head)
    for t, n in zip(secs, lengths):
        if n:
            img[off: off + n].copy_(t)
        off += n
    device_crc32(img, total, img[total:])
    return img


def to_bytes(packed: QuantizedTensor) -> bytes:
    """kvpack.py:126-177: byte-identical serialisation, assembled and
    checksummed on the GPU, then one device->host copy."""
    return to_device_image(packed).cpu().numpy().tobytes()


def write_kvpack(packed: QuantizedTensor, sink) -> int:
    blob = to_bytes(packed)
    if hasattr(sink, "write"):
        sink.write(blob)
    else:
        with open(sink, "wb") as f:
            f.write(blob)
    return len(blob)


def read_kvpack(source, device="cuda") -> QuantizedTensor:
    if hasattr(source, "read"):
        blob = source.read()
    else:
        with open(source, "rb") as f:
            blob = f.read()
    return from_bytes(blob, device)


def from_bytes(blob: bytes, device="cuda") -> QuantizedTensor:
    """Parse and validate (kvpack.py:194-306) with the reference's checks in the
    reference's order.  The file is uploaded once; the CRC-32 is verified on
    the GPU and the sections are carved out of the device copy."""
    import torch

    if len(blob) < HEADER_BYTES + 4:
        raise CorruptData(f"file too short ({len(blob)} bytes)")
    (magic, version, flags, batch, heads, tokens, head_dim, size, radius_bits, role_tag,
     head_base, seed, fixed_mult, layer) = struct.unpack_from(_HEADER_FMT, blob, 0)
    if magic != MAGIC:
        raise CorruptData(f"bad magic {magic!r}")
    if version != VERSION:
        raise UnsupportedVersion(f"format version {version}, expected {VERSION}")
    nat.require_cuda(device)
    device = torch.device(device)
    dblob = torch.frombuffer(bytearray(blob), dtype=torch.uint8).to(device)
    crc = torch.empty(4, dtype=torch.uint8, device=device)
    device_crc32(dblob, len(blob) - 4, crc)
    if bytes(crc.cpu().numpy().tobytes()) != bytes(blob[-4:]):
        raise CorruptData("checksum mismatch")
    table = []
    end = HEADER_BYTES
    for k in range(_SECTION_COUNT):
        off, length = struct.unpack_from("<QQ", blob, 48 + 16 * k)
        if off != end:
            raise CorruptData(f"section {k} offset {off} != expected {end}")
        end = off + length
        table.append((off, length))
    if end + 4 != len(blob):
        raise CorruptData(f"file length {len(blob)} != sections end {end} + checksum")
    roles = {tag: role for role, tag in ROLE_TAGS.items()}
    if role_tag not in roles:
        raise CorruptData(f"unknown role tag {role_tag:#x}")
    outlier = bool(flags & _FLAG_OUTLIER)
    if outlier != (fixed_mult != 0):
        raise CorruptData("outlier flag and multiplier field disagree")
    try:
        shape = TensorShape(batch, heads, tokens, head_dim)
        config = CodecConfig(codebook_size=size, radius_bits=radius_bits, seed=seed,
                             outlier_multiplier=fixed_mult / 65536.0 if outlier else None,
                             median_pooling="per_head" if flags & _FLAG_PER_HEAD else "batch")
    except InvalidArgument as exc:
        raise CorruptData(f"invalid header fields: {exc}") from exc

    def section(k):
        off, length = table[k]
        return blob[off:off + length]

    def dsection(k, nbytes_alloc):
        """Device copy of section k into a zeroed, 4-byte aligned uint8 buffer."""
        off, length = table[k]
        buf = torch.zeros(max(nbytes_alloc, length, 4), dtype=torch.uint8, device=device)
        if length:
            buf[:length].copy_(dblob[off:off + length])
        return buf

    n_tok = batch * heads * tokens
    n = n_tok * shape.chunks_per_vector
    if len(section(0)) != 2 * n_tok:
        raise CorruptData("scale section has the wrong length")
    scales = dsection(0, 2 * n_tok)[: 2 * n_tok].view(torch.float16).reshape(batch, heads, tokens)
    if outlier:
        if len(section(3)) != (n + 7) // 8:
            raise CorruptData("flag bitmap has the wrong length")
        fbits = np.unpackbits(np.frombuffer(section(3), dtype=np.uint8), bitorder="little",
                              count=n)
        n_flag = int(fbits.sum())
        fw = dsection(3, 4 * _words(n)).view(torch.int32)
    else:
        if len(section(3)) != 0:
            raise CorruptData("unexpected flag bitmap without extraction")
        n_flag = 0
        fw = None
    n_coded = n - n_flag
    w, br = config.index_bits, config.radius_bits
    if len(section(1)) != (n_coded * w + 7) // 8:
        raise CorruptData(f"bit stream length {len(section(1))} != expected {(n_coded * w + 7) // 8}")
    if len(section(2)) != (n_coded * br + 7) // 8:
        raise CorruptData(f"bit stream length {len(section(2))} != expected {(n_coded * br + 7) // 8}")
    iw = dsection(1, 4 * _words(n * w)).view(torch.int32)
    rw = dsection(2, 4 * _words(n * br)).view(torch.int32)
    pay_raw = section(4)
    if len(pay_raw) != 8 * n_flag:
        raise CorruptData("payload section has the wrong length")
    # two spare rows: the Med3x decode stages payload rows in 16-byte units
    pay = dsection(4, 8 * (n_flag + 2))[: 8 * (n_flag + 2)].view(torch.float16).reshape(
        n_flag + 2, CHUNK_DIM)
    L = nat.lib()
    tok = None
    if outlier:
        tok = torch.zeros(max(1, n_tok), dtype=torch.int32, device=device)
        ws = torch.empty(int(L.hqmq_token_offsets_workspace_bytes(n_tok)), dtype=torch.uint8,
                         device=device)
        nat.launch(device, "hqmq_token_offsets", L.hqmq_token_offsets, n_tok,
                   shape.chunks_per_vector, fw.data_ptr(), tok.data_ptr(), ws.data_ptr(), ws.numel())
    err = torch.zeros(1, dtype=torch.int32, device=device)
    nat.launch(device, "hqmq_validate_indices", L.hqmq_validate_indices, iw.data_ptr(), n_coded,
               w, config.index_count, err.data_ptr())
    if int(err.item()) & nat.DEVERR_INDEX:
        raise CorruptData("codeword index out of range")
    meta = torch.tensor([n_coded, n_flag, 0, 0], dtype=torch.int64, device=device)
    return QuantizedTensor(shape, config, layer, roles[role_tag], head_base, scales, iw, rw, fw,
                           pay, tok, meta, device, n_coded=n_coded, n_payload=n_flag)


# ------------------------------------------------------------ raw tensors
RAW_MAGIC = b"KVRW"
_RAW_FMT = "<4sBIIII"
_RAW_DTYPES = {0: np.float32, 1: np.float16}


def write_raw(data, sink, dtype: str = "f32") -> int:
    """Dense (batch, heads, tokens, head_dim) tensor file (kvpack.py:309-325):
    header <4sBIIII> (magic, dtype code 0=f32 / 1=f16, shape), row-major body."""
    codes = {"f32": 0, "f16": 1}
    if dtype not in codes:
        raise InvalidArgument(f"dtype must be f32 or f16, got {dtype!r}")
    try:
        import torch

        if torch.is_tensor(data):
            data = data.detach().cpu().numpy()
    except ImportError:  # pragma: no cover
        pass
    data = np.asarray(data)
    if data.ndim != 4:
        raise InvalidArgument("raw tensors must be 4-d (batch, heads, tokens, head_dim)")
    blob = struct.pack(_RAW_FMT, RAW_MAGIC, codes[dtype], *data.shape) + np.ascontiguousarray(
        data.astype(np.dtype(_RAW_DTYPES[codes[dtype]]).newbyteorder("<"))).tobytes()
    if hasattr(sink, "write"):
        sink.write(blob)
    else:
        with open(sink, "wb") as f:
            f.write(blob)
    return len(blob)


def read_raw(source) -> np.ndarray:
    """kvpack.py:328-347, same validation and exceptions."""
    if hasattr(source, "read"):
        blob = source.read()
    else:
        with open(source, "rb") as f:
            blob = f.read()
    head = struct.calcsize(_RAW_FMT)
    if len(blob) < head:
        raise CorruptData("raw tensor file too short")
    magic, code, b, h, t, d = struct.unpack_from(_RAW_FMT, blob, 0)
    if magic != RAW_MAGIC:
        raise CorruptData(f"bad raw magic {magic!r}")
    if code not in _RAW_DTYPES:
        raise CorruptData(f"unknown raw dtype code {code}")
    dt = np.dtype(_RAW_DTYPES[code]).newbyteorder("<")
    expected = head + b * h * t * d * dt.itemsize
    if len(blob) != expected:
        raise CorruptData(f"raw length {len(blob)} != expected {expected}")
    return np.frombuffer(blob[head:], dtype=dt).reshape(b, h, t, d).copy()
