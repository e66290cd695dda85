"""HQMQ codec API on B200: encode/decode of KV tensors through the sm_100a kernels.

Mirrors the reference quantizer API (codec.py:49-349): TensorShape,
CodecConfig, QuantizedTensor, encode_tensor, decode_tensor,
decode_token_range and quantize_dequantize keep their names, argument
meaning, validation and exception types.  What changes is where the data
lives: inputs may be torch tensors (any device) or numpy arrays, and the
QuantizedTensor holds the compressed cache in HBM in its packed form — the
five kvpack sections (kvpack.py:134-146) plus per-token coded offsets — which
is what the decode and fused-attention kernels read.  The reference's dense
views (indices / quanta / flags / payloads, codec.py:124-147) are produced on
demand by the unpack kernel and are read-only snapshots.

No CPU fallback exists: without the C-ABI library or a CUDA device every
entry point raises NativeLibraryMissing.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .codebook import ROLE_TAGS, CodebookBank, effective_size
from .errors import CorruptData, InvalidArgument

CHUNK_DIM = 4
MEDIAN_POOLING_MODES = ("batch", "per_head")
MIN_BITS = 1
MAX_BITS = 8


@dataclass(frozen=True)
class TensorShape:
    """codec.py:49-72."""

    batch: int
    heads: int
    tokens: int
    head_dim: int

    def __post_init__(self):
        if self.batch < 1 or self.heads < 1 or self.head_dim < 1:
            raise InvalidArgument(f"degenerate tensor shape {self}")
        if self.tokens < 0:
            raise InvalidArgument("token count must be nonnegative")

    @property
    def chunks_per_vector(self) -> int:
        return -(-self.head_dim // CHUNK_DIM)

    @property
    def padded_dim(self) -> int:
        return self.chunks_per_vector * CHUNK_DIM

    @property
    def elements(self) -> int:
        return self.batch * self.heads * self.tokens * self.head_dim

    @property
    def n_chunks(self) -> int:
        return self.batch * self.heads * self.tokens * self.chunks_per_vector


@dataclass(frozen=True)
class CodecConfig:
    """codec.py:75-113 (same fields, defaults and validation)."""

    codebook_size: int
    radius_bits: int
    seed: int = 0
    outlier_multiplier: float | None = None
    median_pooling: str = "batch"

    def __post_init__(self):
        if self.codebook_size < 1:
            raise InvalidArgument("codebook size must be >= 1")
        if not 0 <= self.seed < 2**64:
            raise InvalidArgument("seed must fit in an unsigned 64-bit word")
        if not MIN_BITS <= self.radius_bits <= MAX_BITS:
            raise InvalidArgument(f"radius bits must be in [{MIN_BITS}, {MAX_BITS}]")
        if self.outlier_multiplier is not None and not self.outlier_multiplier > 0:
            raise InvalidArgument("outlier multiplier must be positive")
        if self.median_pooling not in MEDIAN_POOLING_MODES:
            raise InvalidArgument(f"median pooling must be one of {MEDIAN_POOLING_MODES}")

    @property
    def index_count(self) -> int:
        return effective_size(self.codebook_size)

    @property
    def index_bits(self) -> int:
        return (self.index_count - 1).bit_length()


def _torch():
    import torch

    return torch


def _dtype_code(dt) -> int:
    torch = _torch()
    return {torch.float16: nat.F16, torch.bfloat16: nat.BF16, torch.float32: nat.F32,
            torch.float64: nat.F64}[dt]


def _words(bits: int) -> int:
    # +4 padding words: the bit reader loads the word after the target and the
    # Med3x TMA decode rounds its bulk copies up to 16 bytes.
    return (bits + 31) // 32 + 4


class QuantizedTensor:
    """Quantized form of one (layer, role) tensor across its heads (codec.py:124-151).

    Device-resident sections: scales (B,H,T) fp16; index/radius bit streams
    (int32 words, LSB-first); flag bitmap (iff extraction); fp16 payload rows;
    per-token coded offsets (iff extraction).
    """

    def __init__(self, shape, config, layer, role, head_base, scales, index_words,
                 radius_words, flag_words, payload_buf, token_offsets, meta, device,
                 n_coded=None, n_payload=None):
        self.shape = shape
        self.config = config
        self.layer = layer
        self.role = role
        self.head_base = head_base
        self.scales = scales
        self.index_words = index_words
        self.radius_words = radius_words
        self.flag_words = flag_words
        self._payload_buf = payload_buf
        self.token_offsets = token_offsets
        self._meta = meta  # int64[4]: n_coded, n_payload, n_fixup, error word
        self.device = device
        self._n_coded = n_coded
        self._n_payload = n_payload
        self._n_fixup = None
        self._dense = None
        self._ready = None  # CUDA event recorded on the encode's stream
        self._ready_stream = None  # ... and that stream's handle
        self._dc = None  # decode fast path: (bank, DecodeArgs template, tables, error word)

    # ------------------------------------------------------------ sync
    def wait(self) -> None:
        """Order the current stream of this tensor's device after the encode
        (a no-op when the encode ran on the same stream or has been waited
        for).  Every device consumer (decode, attention, packing, append)
        calls it first."""
        ev = self._ready
        if ev is not None:
            s = _torch().cuda.current_stream(self.device)
            if s.cuda_stream != self._ready_stream:
                s.wait_event(ev)

    def synchronize(self) -> "QuantizedTensor":
        """Wait for the encode, read its counters and raise its errors."""
        if self._n_coded is None:
            if self._ready is not None:
                self._ready.synchronize()
                self._ready = None  # complete: later consumers need no ordering
            meta = self._meta.cpu().tolist()
            self._n_coded, self._n_payload, self._n_fixup = int(meta[0]), int(meta[1]), int(meta[2])
            err = int(meta[3]) & 0xFFFFFFFF
            if err & nat.DEVERR_SIGMA:
                raise InvalidArgument("sigma must be positive")
            if err & nat.DEVERR_INDEX:
                raise CorruptData("codeword index out of range")
        return self

    @property
    def n_coded(self) -> int:
        return self.synchronize()._n_coded

    @property
    def n_payload(self) -> int:
        return self.synchronize()._n_payload

    @property
    def n_fixup(self) -> int:
        """Chunks the exact fp64 fixup re-scored (diagnostic)."""
        self.synchronize()
        return self._n_fixup or 0

    @property
    def payloads(self):
        return self._payload_buf[: self.n_payload]

    @property
    def outlier_thresholds(self):
        """(G,) float64 device tensor of the Med3x thresholds C * median the
        encode flagged against (G = heads with per-head pooling, else 1), or
        None without extraction."""
        thr = self.__dict__.get("_thresholds")
        if thr is not None:
            self.wait()
        return thr

    @property
    def outlier_fraction(self) -> float:
        n = self.shape.n_chunks
        return self.n_payload / n if n else 0.0

    # ------------------------------------------------------- dense views
    def _unpack(self):
        if self._dense is None:
            torch = _torch()
            s = self.shape
            grid = (s.batch, s.heads, s.tokens, s.chunks_per_vector)
            idx = torch.zeros(grid, dtype=torch.int32, device=self.device)
            q = torch.zeros(grid, dtype=torch.uint8, device=self.device)
            fl = torch.zeros(grid, dtype=torch.uint8, device=self.device)
            if s.n_chunks:
                self.wait()
                args = self._decode_args(0, s.tokens, nat.F32, None, None, None, None)
                nat.launch(self.device, "hqmq_unpack", nat.lib().hqmq_unpack, ctypes.byref(args),
                           idx.data_ptr(), q.data_ptr(), fl.data_ptr())
            self._dense = (idx, q, fl.bool())
        return self._dense

    @property
    def indices(self):
        return self._unpack()[0].clone()

    @property
    def quanta(self):
        return self._unpack()[1].clone()

    @property
    def flags(self):
        return self._unpack()[2].clone()

    # ----------------------------------------------------------- kernels
    def _decode_args(self, start, stop, out_dtype, out, err, j32, j64, j16=None):
        s, c = self.shape, self.config
        a = nat.DecodeArgs()
        a.batch, a.heads, a.tokens, a.head_dim = s.batch, s.heads, s.tokens, s.head_dim
        a.codebook_size, a.radius_bits, a.index_bits = c.codebook_size, c.radius_bits, c.index_bits
        a.out_dtype = out_dtype
        a.token_start, a.token_stop = start, stop
        a.scales = self.scales.data_ptr()
        a.index_words = self.index_words.data_ptr()
        a.radius_words = self.radius_words.data_ptr()
        a.flag_words = self.flag_words.data_ptr() if self.flag_words is not None else None
        a.payloads = self._payload_buf.data_ptr() if self.flag_words is not None else None
        a.token_offsets = self.token_offsets.data_ptr() if self.token_offsets is not None else None
        a.joint_f32 = j32.data_ptr() if j32 is not None else None
        a.joint_f64 = j64.data_ptr() if j64 is not None else None
        a.joint_f16 = j16.data_ptr() if j16 is not None else None
        a.out = out.data_ptr() if out is not None else None
        a.error_word = err.data_ptr() if err is not None else None
        return a

    def packed_view(self, bank: CodebookBank) -> nat.PackedView:
        self.wait()
        pv = self.__dict__.get("_pv")
        if pv is not None and pv[0] is bank:
            return pv[1]
        tabs = bank.device_tables(self.layer, self.head_base, self.shape.heads, self.role,
                                  self.device)
        v = nat.PackedView()
        v.scales = self.scales.data_ptr()
        v.index_words = self.index_words.data_ptr()
        v.radius_words = self.radius_words.data_ptr()
        v.flag_words = self.flag_words.data_ptr() if self.flag_words is not None else None
        v.payloads = self._payload_buf.data_ptr() if self.flag_words is not None else None
        v.token_offsets = self.token_offsets.data_ptr() if self.token_offsets is not None else None
        v.joint_f32 = tabs["joint_f32"].data_ptr()
        v.joint_f16 = tabs["joint_f16"].data_ptr()
        v.joint_f64 = tabs["joint_f64"].data_ptr()
        self._pv = (bank, v, tabs)
        return v

    # ---------------------------------------------------------- sections
    def section_bytes(self) -> list:
        """The five kvpack sections (kvpack.py:134-146) as bytes."""
        s, c = self.shape, self.config
        n_coded = self.n_coded
        scales = self.scales.contiguous().cpu().numpy().astype("<f2").tobytes()

        def stream(words, width):
            nbytes = (n_coded * width + 7) // 8
            raw = words.cpu().numpy().astype("<u4").tobytes()
            return raw[:nbytes]

        idx = stream(self.index_words, c.index_bits)
        rad = stream(self.radius_words, c.radius_bits)
        if c.outlier_multiplier is not None:
            fl = self.flag_words.cpu().numpy().astype("<u4").tobytes()[: (s.n_chunks + 7) // 8]
        else:
            fl = b""
        pay = self.payloads.contiguous().cpu().numpy().astype("<f2").tobytes()
        return [scales, idx, rad, fl, pay]

    # -------------------------------------------------------- construct
    @classmethod
    def from_arrays(cls, shape: TensorShape, config: CodecConfig, layer: int, role: str,
                    scales, indices, quanta, flags, payloads, head_base: int = 0,
                    device="cuda") -> "QuantizedTensor":
        """Pack dense arrays (the reference's QuantizedTensor fields) into sections."""
        torch = _torch()
        nat.require_cuda(device)
        device = torch.device(device)
        s, c = shape, config
        n = s.n_chunks
        grid = (s.batch, s.heads, s.tokens, s.chunks_per_vector)
        to = lambda a, dt: torch.as_tensor(np.asarray(a) if not torch.is_tensor(a) else a).to(
            device=device, dtype=dt).contiguous()
        idx = to(indices, torch.int32).reshape(grid)
        q = to(quanta, torch.uint8).reshape(grid)
        ext = c.outlier_multiplier is not None
        fl = to(flags, torch.uint8).reshape(grid) if ext else None
        if idx.numel() and (int(idx.min()) < 0 or int(idx.max()) >= c.index_count):
            raise CorruptData("codeword index out of range")
        n_flag = int(fl.sum()) if ext else 0
        iw = torch.zeros(_words(n * c.index_bits), dtype=torch.int32, device=device)
        rw = torch.zeros(_words(n * c.radius_bits), dtype=torch.int32, device=device)
        fw = torch.zeros(_words(n), dtype=torch.int32, device=device) if ext else None
        tok = torch.zeros(max(1, s.batch * s.heads * s.tokens), dtype=torch.int32,
                          device=device) if ext else None
        ws = torch.empty(int(nat.lib().hqmq_pack_workspace_bytes(n)), dtype=torch.uint8,
                         device=device)
        nat.launch(device, "hqmq_pack", nat.lib().hqmq_pack,
                   n, s.chunks_per_vector, c.index_bits, c.radius_bits, idx.data_ptr(), q.data_ptr(),
                   fl.data_ptr() if ext else None, iw.data_ptr(), rw.data_ptr(),
                   fw.data_ptr() if ext else None, tok.data_ptr() if ext else None,
                   ws.data_ptr(), ws.numel())
        sc = torch.as_tensor(np.asarray(scales, dtype=np.float16) if not torch.is_tensor(scales)
                             else scales).to(device=device, dtype=torch.float16).reshape(
                                 s.batch, s.heads, s.tokens).contiguous()
        pay = torch.as_tensor(np.asarray(payloads, dtype=np.float16) if not torch.is_tensor(payloads)
                              else payloads).to(device=device, dtype=torch.float16).reshape(-1, 4)
        if pay.shape[0] != n_flag:
            raise CorruptData("payload count does not match the flags")
        pay_buf = torch.zeros((n_flag + 2, 4), dtype=torch.float16, device=device)
        pay_buf[:n_flag] = pay
        meta = torch.tensor([n - n_flag, n_flag, 0, 0], dtype=torch.int64, device=device)
        return cls(s, c, layer, role, head_base, sc, iw, rw, fw, pay_buf, tok, meta, device,
                   n_coded=n - n_flag, n_payload=n_flag)

    @classmethod
    def from_reference(cls, packed, device="cuda") -> "QuantizedTensor":
        """Wrap a reference (numpy) QuantizedTensor, e.g. hqmq.codec.QuantizedTensor."""
        rs, rc = packed.shape, packed.config
        shape = TensorShape(rs.batch, rs.heads, rs.tokens, rs.head_dim)
        config = CodecConfig(rc.codebook_size, rc.radius_bits, rc.seed, rc.outlier_multiplier,
                             rc.median_pooling)
        return cls.from_arrays(shape, config, packed.layer, packed.role, packed.scales,
                               packed.indices, packed.quanta, packed.flags, packed.payloads,
                               packed.head_base, device)


# --------------------------------------------------------------- helpers
def same_device(a, b) -> bool:
    """torch.device equality with an index-less 'cuda' meaning the current device."""
    if a == b:
        return True
    torch = _torch()
    a, b = torch.device(a), torch.device(b)
    if a.type != b.type:
        return False
    if a.type != "cuda":
        return True
    cur = torch.cuda.current_device()
    return (a.index if a.index is not None else cur) == (b.index if b.index is not None else cur)


def check_out(out, shape, dtype, device, what: str = "out") -> None:
    """A caller-supplied output buffer must be exactly what the kernel writes:
    a contiguous CUDA tensor of this shape and dtype on the packed tensor's
    device (the kernels write a dense block at out.data_ptr())."""
    torch = _torch()
    if not torch.is_tensor(out):
        raise InvalidArgument(f"{what} must be a torch tensor")
    if out.dtype != dtype:
        raise InvalidArgument(f"{what} has dtype {out.dtype}, expected {dtype}")
    if tuple(out.shape) != tuple(shape):
        raise InvalidArgument(f"{what} has shape {tuple(out.shape)}, expected {tuple(shape)}")
    if not out.is_cuda or (out.device != device and not same_device(out.device, device)):
        raise InvalidArgument(f"{what} must live on {device}, got {out.device}")
    if not out.is_contiguous():
        raise InvalidArgument(f"{what} must be contiguous")


def _bank_for(config: CodecConfig, bank: CodebookBank | None) -> CodebookBank:
    """codec.py:222-229."""
    if bank is None:
        return CodebookBank(seed=config.seed, size=config.codebook_size)
    if bank.seed != config.seed or bank.size != config.codebook_size:
        raise InvalidArgument("codebook bank does not match the codec config (seed or size)")
    return bank


def _as_device_4d(data, device):
    torch = _torch()
    if not torch.is_tensor(data):
        arr = np.asarray(data)
        if arr.dtype not in (np.float16, np.float32, np.float64):
            arr = arr.astype(np.float64)
        data = torch.from_numpy(np.ascontiguousarray(arr))
    if data.dtype not in (torch.float16, torch.bfloat16, torch.float32, torch.float64):
        data = data.to(torch.float64)
    if data.dim() != 4:
        raise InvalidArgument(f"expected (batch, heads, tokens, head_dim) data, got ndim={data.dim()}")
    nat.require_cuda(device)
    if device is None:
        device = data.device if data.is_cuda else torch.device("cuda", torch.cuda.current_device())
    device = torch.device(device)
    if device.index is None:
        device = torch.device("cuda", torch.cuda.current_device())
    data = data.to(device=device, non_blocking=True).contiguous()
    return data, TensorShape(*data.shape), device


SEARCH_PATHS = {"auto": nat.SEARCH_AUTO, "cuda_core": nat.SEARCH_CUDA_CORE,
                "tensor_core": nat.SEARCH_TENSOR_CORE}


def encode_tensor(data, config: CodecConfig, layer: int = 0, role: str = "K",
                  bank: CodebookBank | None = None, head_base: int = 0, *,
                  device=None, sync: bool = True, search_path: str = "auto",
                  outlier_thresholds=None) -> QuantizedTensor:
    """Quantize a (batch, heads, tokens, head_dim) tensor (codec.py:232-287).

    Runs Med3x, the fused encode kernel and the section packing on the GPU.
    sync=True (reference semantics) waits for the kernels and raises
    InvalidArgument on a non-positive scale; sync=False returns immediately and
    defers that check to QuantizedTensor.synchronize().  search_path selects
    the nearest-codeword search of the fp16/bf16 head_dim-128 kernels
    ("auto", "cuda_core" = FFMA2, "tensor_core" = tcgen05 rotations when
    S % 16 == 0); every path is certified and bit-identical to the reference.

    outlier_thresholds (extension, Med3x only): freeze the outlier thresholds
    instead of pooling this call's median -- a float or a (G,) float64 tensor,
    G = heads with per-head pooling else 1; chunks with r > threshold are
    extracted (the reference's strict test, codec.py:208-219, against a given
    threshold).  The thresholds an encode used are on
    QuantizedTensor.outlier_thresholds, so a cache's prefill encode can freeze
    them for its appends (PagedKVCache).
    """
    torch = _torch()
    if role not in ROLE_TAGS:
        raise InvalidArgument(f"role must be one of {sorted(ROLE_TAGS)}")
    if search_path not in SEARCH_PATHS:
        raise InvalidArgument(f"search_path must be one of {sorted(SEARCH_PATHS)}")
    if head_base < 0:
        raise InvalidArgument("head_base must be nonnegative")
    data, shape, device = _as_device_4d(data, device)
    bank = _bank_for(config, bank)
    c = config
    n = shape.n_chunks
    ext = c.outlier_multiplier is not None
    rows_t = shape.batch * shape.heads * shape.tokens
    scales = torch.empty((shape.batch, shape.heads, shape.tokens), dtype=torch.float16,
                         device=device)
    iw = torch.empty(_words(n * c.index_bits), dtype=torch.int32, device=device)
    rw = torch.empty(_words(n * c.radius_bits), dtype=torch.int32, device=device)
    fw = torch.empty(_words(n), dtype=torch.int32, device=device) if ext else None
    tok = torch.empty(max(1, rows_t), dtype=torch.int32, device=device) if ext else None
    if ext:
        groups = shape.heads if c.median_pooling == "per_head" else 1
        cap = n // 2 + groups + 1 if c.outlier_multiplier >= 1.0 else n + 1
    else:
        cap = 1
    pay = torch.empty((cap, 4), dtype=torch.float16, device=device)
    meta = torch.empty(4, dtype=torch.int64, device=device)  # zeroed by hqmq_encode
    thr_out = fixed = None
    if ext:
        G = shape.heads if c.median_pooling == "per_head" else 1
        thr_out = torch.empty(G, dtype=torch.float64, device=device)
        if outlier_thresholds is not None:
            fixed = torch.as_tensor(outlier_thresholds, dtype=torch.float64)
            fixed = (fixed.reshape(1).expand(G) if fixed.numel() == 1 else fixed.reshape(-1))
            if fixed.numel() != G:
                raise InvalidArgument(f"outlier_thresholds needs {G} values, got {fixed.numel()}")
            fixed = fixed.to(device=device).contiguous()
    elif outlier_thresholds is not None:
        raise InvalidArgument("outlier_thresholds requires outlier extraction (outlier_multiplier)")
    tabs = bank.device_tables(layer, head_base, shape.heads, role, device)
    a = nat.EncodeArgs()
    a.batch, a.heads, a.tokens, a.head_dim = shape.batch, shape.heads, shape.tokens, shape.head_dim
    a.codebook_size, a.radius_bits, a.index_bits = c.codebook_size, c.radius_bits, c.index_bits
    a.input_dtype = _dtype_code(data.dtype)
    a.outlier_multiplier = float(c.outlier_multiplier) if ext else 0.0
    a.per_head_pooling = 1 if c.median_pooling == "per_head" else 0
    a.data = data.data_ptr()
    a.rot_f32 = tabs["rot_f32"].data_ptr()
    a.joint_f64 = tabs["joint_f64"].data_ptr()
    a.scales = scales.data_ptr()
    a.index_words, a.radius_words = iw.data_ptr(), rw.data_ptr()
    a.flag_words = fw.data_ptr() if ext else None
    a.payloads = pay.data_ptr()
    a.token_offsets = tok.data_ptr() if ext else None
    a.payload_capacity = cap if ext else 0
    a.counters = meta.data_ptr()
    a.error_word = meta.data_ptr() + 24
    a.index_capacity_words, a.radius_capacity_words = iw.numel(), rw.numel()
    a.search_path = SEARCH_PATHS[search_path]
    a.flag_capacity_words = fw.numel() if ext else 0
    a.fixed_thresholds = fixed.data_ptr() if fixed is not None else None
    a.thresholds_out = thr_out.data_ptr() if thr_out is not None else None
    L = nat.lib()
    ws_bytes = int(L.hqmq_encode_workspace_bytes(ctypes.byref(a)))
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=device) if ws_bytes else None
    a.workspace, a.workspace_bytes = (ws.data_ptr() if ws is not None else None), ws_bytes
    nat.launch(device, "hqmq_encode", L.hqmq_encode, ctypes.byref(a))
    qt = QuantizedTensor(shape, config, layer, role, head_base, scales, iw, rw, fw, pay, tok,
                         meta, device)
    qt._keepalive = (data, ws, fixed)
    qt._thresholds = thr_out
    st = torch.cuda.current_stream(device)
    qt._ready = torch.cuda.Event()
    qt._ready.record(st)
    qt._ready_stream = st.cuda_stream
    if sync:
        qt.synchronize()
    return qt


_OUT_CODES = {}


def _out_code(dtype):
    if not _OUT_CODES:
        torch = _torch()
        _OUT_CODES.update({torch.float32: nat.F32, torch.float16: nat.F16,
                           torch.bfloat16: nat.BF16, torch.float64: nat.F64})
    code = _OUT_CODES.get(dtype)
    if code is None:
        raise InvalidArgument("decode dtype must be float16, bfloat16, float32 or float64")
    return code


def decode_token_range(packed: QuantizedTensor, bank: CodebookBank, start: int, stop: int,
                       dtype=None, *, out=None, check: bool = True):
    """Decode tokens [start, stop) to a dense (B, H, stop-start, head_dim) tensor
    (codec.py:290-328).  dtype float64 is bit-identical to the reference;
    float32 (default) is within 1e-6 relative; float16/bfloat16 for serving."""
    torch = _torch()
    if dtype is None:
        dtype = out.dtype if out is not None else torch.float32
    s = packed.shape
    if not 0 <= start <= stop <= s.tokens:
        raise InvalidArgument(f"token range [{start}, {stop}) out of bounds")
    code = _out_code(dtype)
    dev = packed.device
    want = (s.batch, s.heads, stop - start, s.head_dim)
    if out is None:
        out = torch.empty(want, dtype=dtype, device=dev)
    else:
        check_out(out, want, dtype, dev, "decode out")
    if stop == start:
        return out
    # per-(tensor, bank) argument block, tables and error word, built once: the
    # error word only accumulates bits (a corrupt index stays corrupt), so it
    # is never reset
    dc = packed._dc
    if dc is None or dc[0] is not bank:
        tabs = bank.device_tables(packed.layer, packed.head_base, s.heads, packed.role, dev)
        # decode index errors OR into the tensor's own error word (meta[3], zeroed by
        # the encode): no allocation or fill per tensor
        err = packed._meta.view(torch.int32)[6:7]
        args = packed._decode_args(0, 0, code, None, err, tabs["joint_f32"], tabs["joint_f64"],
                                   tabs["joint_f16"])
        dc = packed._dc = (bank, args, tabs, err)
    args, err = dc[1], dc[3]
    args.token_start, args.token_stop, args.out_dtype = start, stop, code
    args.out = out.data_ptr()
    packed.wait()
    nat.launch(dev, "hqmq_decode", nat.lib().hqmq_decode, ctypes.byref(args))
    if check and int(err.item()) & nat.DEVERR_INDEX:
        raise CorruptData("codeword index out of range")
    return out


def decode_tensor(packed: QuantizedTensor, bank: CodebookBank | None = None, dtype=None, *,
                  out=None, check: bool = True):
    """Reconstruct the full (batch, heads, tokens, head_dim) tensor (codec.py:331-336)."""
    bank = _bank_for(packed.config, bank)
    return decode_token_range(packed, bank, 0, packed.shape.tokens, dtype, out=out, check=check)


def quantize_dequantize(data, config: CodecConfig, layer: int = 0, role: str = "K",
                        bank: CodebookBank | None = None, head_base: int = 0, dtype=None):
    """Fake-quant round trip (codec.py:339-349)."""
    bank = _bank_for(config, bank)
    return decode_tensor(encode_tensor(data, config, layer, role, bank, head_base), bank, dtype)


def append_tokens(packed: QuantizedTensor, data, bank: CodebookBank | None = None) -> QuantizedTensor:
    """Grow a compressed cache along the token axis:
    encode `data` (batch, heads, new_tokens, head_dim) with the cache's config,
    layer, role and head_base, and return the concatenated QuantizedTensor.

    Without Med3x the encode is token-local (codec.py:258-274: sigma per token,
    index per chunk), so the result is bit-identical to encode_tensor of the
    concatenated input, and every token's codes occupy whole 32-bit words: the
    append is the sm_100a encode of the new tokens plus row-strided device
    copies of the sections.  With Med3x the reference pools the median over the
    whole call (codec.py:208-219), so an exact append needs the full input;
    that case raises InvalidArgument.
    """
    torch = _torch()
    c, s = packed.config, packed.shape
    if c.outlier_multiplier is not None:
        raise InvalidArgument("append_tokens with outlier extraction: the Med3x median pools the "
                              "whole call, re-encode the full tensor instead")
    bank = _bank_for(c, bank)
    new = encode_tensor(data, c, layer=packed.layer, role=packed.role, bank=bank,
                        head_base=packed.head_base, device=packed.device)
    ns = new.shape
    if (ns.batch, ns.heads, ns.head_dim) != (s.batch, s.heads, s.head_dim):
        raise InvalidArgument(f"appended data {tuple((ns.batch, ns.heads, ns.tokens, ns.head_dim))} "
                              f"does not match the cache {tuple((s.batch, s.heads, s.tokens, s.head_dim))}")
    shape = TensorShape(s.batch, s.heads, s.tokens + ns.tokens, s.head_dim)
    rows, C = s.batch * s.heads, s.chunks_per_vector
    dev = packed.device

    def cat_words(old, fresh, width):
        per_tok = C * width  # bits per token
        if per_tok % 32:
            raise InvalidArgument("token codes are not word-aligned for this head_dim / width")
        wpt = per_tok // 32
        out = torch.zeros(_words(shape.n_chunks * width), dtype=torch.int32, device=dev)
        dst = out[: rows * shape.tokens * wpt].view(rows, shape.tokens * wpt)
        dst[:, : s.tokens * wpt].copy_(old[: rows * s.tokens * wpt].view(rows, s.tokens * wpt))
        dst[:, s.tokens * wpt:].copy_(fresh[: rows * ns.tokens * wpt].view(rows, ns.tokens * wpt))
        return out

    new.synchronize()
    packed.wait()
    iw = cat_words(packed.index_words, new.index_words, c.index_bits)
    rw = cat_words(packed.radius_words, new.radius_words, c.radius_bits)
    scales = torch.cat([packed.scales, new.scales], dim=2).contiguous()
    n = shape.n_chunks
    meta = torch.tensor([n, 0, packed.n_fixup + new.n_fixup, 0], dtype=torch.int64, device=dev)
    pay = torch.zeros((1, 4), dtype=torch.float16, device=dev)
    return QuantizedTensor(shape, c, packed.layer, packed.role, packed.head_base, scales, iw, rw,
                           None, pay, None, meta, dev, n_coded=n, n_payload=0)
