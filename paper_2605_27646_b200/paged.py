"""Paged HQMQ KV cache for decode-time serving (append
encode into a paged layout; north star: decode fused inside a *paged*
decode-attention kernel).

The reference keeps one dense tensor per (layer, role) and has no append
(codec.py:232-287).  Here a cache for one layer holds K and V as pools of
128-token pages; a page is one (sequence, kv head) row's tokens
[128 i, 128 i + 128) in fixed per-token code slots (index_bits words of index
codes, radius_bits words of radius codes and one fp16 scale per token), so
appending is:

  1. encode_tensor of the new tokens (the sm_100a encode, bit-identical to the
     reference on those tokens: without extraction the codec is token-local);
  2. one scatter kernel per role (hqmq_paged_append) moving each new token's
     code words, scale (and Med3x flag word / payload offset) into its page
     slot, the slot computed on the device from the block table; pages are
     taken from a free list as rows grow.

attend() runs the decode-attention kernel with a block table
(hqmq_attention_decode_paged).

Med3x (outlier_multiplier set).  The reference pools the median over the
whole (layer, role) call (codec.py:208-219; outliers.py:50-55) and has no
incremental form (PAPER.md:138 names an EMA or frozen median as the options).
This cache uses a FROZEN threshold: the first append of each role (the
prefill) is encoded exactly as the reference's encode_tensor of that call --
its own C * lower median, bit-identical -- and its thresholds
(QuantizedTensor.outlier_thresholds; one per head with per-head pooling) are
kept; every later append flags chunks with r > that frozen threshold (the
reference's strict test) instead of re-pooling.  Deviation from a one-shot
encode of the concatenation: appended tokens are flagged against the prefill's
median rather than the median of everything cached so far.  The appended
encode is then token-local (appending tokens one by one equals appending them
at once) and bit-exact against the oracle's encode with the same thresholds.
Thresholds can also be given up front (outlier_thresholds=).  Storage: each
token keeps its fixed code slots (a flagged chunk's slot is 0), a 32-bit flag
word and the row of its first payload in a per-role fp16 payload pool
(hqmq_expand_tokens converts the encoder's compact sections).
"""

from __future__ import annotations

import ctypes
import math

from . import _native as nat
from .codebook import CodebookBank
from .codec import CodecConfig, _bank_for, _torch, check_out, encode_tensor
from .errors import CorruptData, InvalidArgument

PAGE_TOKENS = 128


class PagedKVCache:
    """K/V page pools of one layer for `batch` sequences of up to `max_tokens`."""

    def __init__(self, config: CodecConfig, batch: int, kv_heads: int, max_tokens: int,
                 layer: int = 0, bank: CodebookBank | None = None, head_base: int = 0,
                 head_dim: int = 128, num_pages: int | None = None, device="cuda",
                 page_order_seed: int | None = None, outlier_thresholds=None):
        torch = _torch()
        self.med3x = config.outlier_multiplier is not None
        if outlier_thresholds is not None and not self.med3x:
            raise InvalidArgument("outlier_thresholds requires outlier extraction")
        if self.med3x and config.codebook_size > 170:
            # the Med3x paged kernel keeps four 24*S-entry fp16 tables (K and V,
            # each with its residual) in shared memory: S <= 170 (index_bits <= 12)
            raise InvalidArgument("paged Med3x caches support codebook_size <= 170")
        if head_dim != 128:
            raise InvalidArgument("paged caches support head_dim 128")
        if batch < 1 or kv_heads < 1 or max_tokens < 1:
            raise InvalidArgument("batch, kv_heads and max_tokens must be positive")
        nat.require_cuda(device)
        self.config, self.layer, self.head_base = config, layer, head_base
        self.bank = _bank_for(config, bank)
        self.batch, self.kv_heads, self.head_dim = batch, kv_heads, head_dim
        self.device = torch.device(device)
        self.max_pages = math.ceil(max_tokens / PAGE_TOKENS)
        self.max_tokens = self.max_pages * PAGE_TOKENS
        rows = batch * kv_heads
        self.num_pages = num_pages if num_pages is not None else rows * self.max_pages
        w, br = config.index_bits, config.radius_bits
        dev = self.device
        self.pages = {}
        for role in ("K", "V"):
            self.pages[role] = {
                # + one spare page: the attention kernels read a few words past a
                # token's codes, also for the last token of the last page
                "index": torch.zeros((self.num_pages + 1, PAGE_TOKENS * w), dtype=torch.int32,
                                     device=dev),
                "radius": torch.zeros((self.num_pages + 1, PAGE_TOKENS * br), dtype=torch.int32,
                                      device=dev),
                "scales": torch.zeros((self.num_pages + 1, PAGE_TOKENS), dtype=torch.float16,
                                      device=dev),
            }
            if self.med3x:
                self.pages[role]["flags"] = torch.zeros((self.num_pages + 1, PAGE_TOKENS),
                                                        dtype=torch.int32, device=dev)
                self.pages[role]["payoff"] = torch.zeros((self.num_pages + 1, PAGE_TOKENS),
                                                         dtype=torch.int32, device=dev)
        # Med3x: per-role fp16 payload pools (rows in use) and frozen thresholds
        self.payloads = {r: torch.zeros((1024, 4), dtype=torch.float16, device=dev)
                         for r in ("K", "V")} if self.med3x else None
        self.n_payload = {"K": 0, "V": 0}
        self.thresholds = {"K": None, "V": None}
        if outlier_thresholds is not None:
            for r in ("K", "V"):
                thr = outlier_thresholds[r] if isinstance(outlier_thresholds, dict) \
                    else outlier_thresholds
                self.thresholds[r] = torch.as_tensor(thr, dtype=torch.float64).reshape(-1).to(dev)
        self.block_table = torch.full((batch, kv_heads, self.max_pages), -1, dtype=torch.int32,
                                      device=dev)
        self._table_host = [[[-1] * self.max_pages for _ in range(kv_heads)] for _ in range(batch)]
        self.lengths = [0] * batch
        self.kv_lens = torch.zeros(batch, dtype=torch.int32, device=dev)
        # device error word of the append scatter (HQMQ_DEVERR_INDEX_RANGE on a
        # page id outside the pool: not reachable through this class's own
        # page bookkeeping; read by check_errors())
        self._err = torch.zeros(1, dtype=torch.int32, device=dev)
        self._free = list(range(self.num_pages - 1, -1, -1))
        if page_order_seed is not None:  # a fragmented pool: pages handed out in random order
            import random

            random.Random(page_order_seed).shuffle(self._free)

    # ------------------------------------------------------------ append
    def _page(self, b: int, h: int, i: int) -> int:
        pid = self._table_host[b][h][i]
        if pid < 0:
            if not self._free:
                raise InvalidArgument("page pool exhausted")
            pid = self._free.pop()
            self._table_host[b][h][i] = pid
        return pid

    def append(self, k, v, seqs=None) -> None:
        """Append new tokens (len(seqs), kv_heads, n_new, head_dim) for the listed
        sequences (default: all, in order)."""
        torch = _torch()
        seqs = list(range(self.batch)) if seqs is None else list(seqs)
        if len(set(seqs)) != len(seqs) or any(not 0 <= b < self.batch for b in seqs):
            raise InvalidArgument(f"seqs must be distinct sequence ids in [0, {self.batch})")
        shape = tuple(k.shape)
        if shape != tuple(v.shape) or len(shape) != 4 or shape[0] != len(seqs) or \
                shape[1] != self.kv_heads or shape[3] != self.head_dim:
            raise InvalidArgument(f"k/v shape {shape} does not match the cache")
        n_new = shape[2]
        if n_new == 0:
            return
        for b in seqs:
            if self.lengths[b] + n_new > self.max_tokens:
                raise InvalidArgument(f"sequence {b} would exceed {self.max_tokens} tokens")
        # take pages for the new tokens, then the destination slot
        # (page * 128 + offset) of every new token in encode order (seq, head, token)
        for b in seqs:
            first, last = self.lengths[b] // PAGE_TOKENS, (self.lengths[b] + n_new - 1) // PAGE_TOKENS
            for h in range(self.kv_heads):
                for i in range(first, last + 1):
                    self._page(b, h, i)
        self.block_table.copy_(torch.tensor(self._table_host, dtype=torch.int32))
        dev = self.device
        # (seq ids, cached lengths) of the appended sequences; the scatter into
        # the page slots is one kernel per role (hqmq_paged_append)
        seq_info = torch.tensor([seqs, [self.lengths[b] for b in seqs]], dtype=torch.int32,
                                device=dev)
        n_tok = len(seqs) * self.kv_heads * n_new
        w, br = self.config.index_bits, self.config.radius_bits
        for role, x in (("K", k), ("V", v)):
            qt = encode_tensor(x, self.config, layer=self.layer, role=role, bank=self.bank,
                               head_base=self.head_base, device=self.device,
                               outlier_thresholds=self.thresholds[role] if self.med3x else None)
            pool = self.pages[role]
            a = nat.PagedAppendArgs()
            a.n_seq, a.kv_heads, a.n_new, a.max_pages = len(seqs), self.kv_heads, n_new, \
                self.max_pages
            a.page_tokens, a.index_bits, a.radius_bits = PAGE_TOKENS, w, br
            a.num_pages = self.num_pages
            a.seq_ids, a.seq_start = seq_info[0].data_ptr(), seq_info[1].data_ptr()
            a.block_table = self.block_table.data_ptr()
            if self.med3x:
                if self.thresholds[role] is None:  # the prefill freezes its thresholds
                    self.thresholds[role] = qt.outlier_thresholds.clone()
                iw, rw, payoff = self._expand(role, qt, n_tok)
                a.src_flags, a.src_payoff = qt.flag_words.data_ptr(), payoff.data_ptr()
                a.flag_pages, a.payoff_pages = pool["flags"].data_ptr(), pool["payoff"].data_ptr()
            else:
                iw, rw = qt.index_words, qt.radius_words
            a.src_index, a.src_radius = iw.data_ptr(), rw.data_ptr()
            a.src_scales = qt.scales.data_ptr()
            a.index_pages, a.radius_pages = pool["index"].data_ptr(), pool["radius"].data_ptr()
            a.scale_pages = pool["scales"].data_ptr()
            a.error_word = self._err.data_ptr()
            nat.launch(dev, "hqmq_paged_append", nat.lib().hqmq_paged_append, ctypes.byref(a))
        for b in seqs:
            self.lengths[b] += n_new
        self.kv_lens.copy_(torch.tensor(self.lengths, dtype=torch.int32))

    def check_errors(self) -> None:
        """Raise CorruptData if an append met a page id outside the pool
        (synchronises with the device)."""
        if int(self._err.item()):
            raise CorruptData("paged append: page id outside the page pool")

    def _expand(self, role, qt, n_tok):
        """Med3x: the encoder's compact sections -> fixed per-token slots and
        payload-row offsets, the payload rows appended to the role's pool
        (hqmq_expand_tokens)."""
        torch = _torch()
        c, dev = self.config, self.device
        n_pay = qt.n_payload
        base = self.n_payload[role]
        if base + n_pay >= 2 ** 32:
            raise InvalidArgument("Med3x payload pool exceeds 2^32 rows")
        pool = self.payloads[role]
        if base + n_pay > pool.shape[0]:  # grow geometrically
            grown = torch.zeros((max(2 * pool.shape[0], base + n_pay), 4), dtype=torch.float16,
                                device=dev)
            grown[:base].copy_(pool[:base])
            self.payloads[role] = pool = grown
        pool[base:base + n_pay].copy_(qt.payloads)
        self.n_payload[role] = base + n_pay
        iw = torch.empty(n_tok * c.index_bits, dtype=torch.int32, device=dev)
        rw = torch.empty(n_tok * c.radius_bits, dtype=torch.int32, device=dev)
        payoff = torch.empty(n_tok, dtype=torch.int32, device=dev)
        args = qt._decode_args(0, qt.shape.tokens, nat.F32, None, None, None, None)
        nat.launch(dev, "hqmq_expand_tokens", nat.lib().hqmq_expand_tokens, ctypes.byref(args),
                   iw.data_ptr(), rw.data_ptr(), payoff.data_ptr(), base)
        return iw, rw, payoff

    # ------------------------------------------------------------ attend
    def attend(self, q, scale: float | None = None, out=None, num_splits: int = 0):
        """One decode step: q (batch, q_heads, 1, head_dim) fp32 -> attention over
        each sequence's cached keys (fused decode, paged block table)."""
        torch = _torch()
        B, HQ, TQ, D = q.shape
        if B != self.batch or TQ != 1 or D != self.head_dim or HQ % self.kv_heads:
            raise InvalidArgument(f"q shape {tuple(q.shape)} does not match the cache")
        if min(self.lengths) == 0:
            raise InvalidArgument("every sequence needs at least one cached token")
        q = q.to(device=self.device, dtype=torch.float32).contiguous()
        if out is None:
            out = torch.empty_like(q)
        else:
            check_out(out, tuple(q.shape), torch.float32, self.device, "attend out")
        c = self.config
        a = nat.PagedAttentionArgs()
        a.batch, a.q_heads, a.kv_heads, a.head_dim = B, HQ, self.kv_heads, D
        a.codebook_size, a.radius_bits, a.index_bits = c.codebook_size, c.radius_bits, c.index_bits
        a.page_tokens, a.max_pages = PAGE_TOKENS, self.max_pages
        a.max_kv_tokens = max(self.lengths)
        a.scale = float(scale if scale is not None else D ** -0.5)
        a.kv_lens, a.block_table = self.kv_lens.data_ptr(), self.block_table.data_ptr()
        a.q, a.out = q.data_ptr(), out.data_ptr()
        for role, view in (("K", a.k), ("V", a.v)):
            tabs = self.bank.device_tables(self.layer, self.head_base, self.kv_heads, role,
                                           self.device)
            pool = self.pages[role]
            view.index_pages = pool["index"].data_ptr()
            view.radius_pages = pool["radius"].data_ptr()
            view.scale_pages = pool["scales"].data_ptr()
            view.joint_f32 = tabs["joint_f32"].data_ptr()
            view.joint_f16 = tabs["joint_f16"].data_ptr()
            if self.med3x:
                view.flag_pages = pool["flags"].data_ptr()
                view.payoff_pages = pool["payoff"].data_ptr()
                view.payloads = self.payloads[role].data_ptr()
        a.num_splits = num_splits
        L = nat.lib()
        ws_bytes = int(L.hqmq_paged_attention_workspace_bytes(ctypes.byref(a)))
        ws = torch.empty(max(1, ws_bytes), dtype=torch.uint8, device=self.device)
        a.workspace, a.workspace_bytes = ws.data_ptr(), ws_bytes
        nat.launch(self.device, "hqmq_attention_decode_paged", L.hqmq_attention_decode_paged,
                   ctypes.byref(a))
        out._ws = ws
        return out
