"""The C-ABI library loads and exports every symbol include/hqmq_b200.h declares.

CPU-only: no compute calls (no GPU here); only host-side queries.
"""

import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "hqmq_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hqmq_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ("hqmq_nearest_scan", "hqmq_encode", "hqmq_decode", "hqmq_unpack",
                     "hqmq_pack", "hqmq_token_offsets", "hqmq_validate_indices",
                     "hqmq_attention_decode"):
        assert required in names


def test_library_exports_every_declared_symbol():
    from paper_2605_27646_b200 import _native

    lib = _native.load()
    for name in declared_functions():
        assert hasattr(lib, name), name
        assert name in _native.SIGNATURES, f"{name} has no ctypes signature"


def test_host_queries():
    from paper_2605_27646_b200 import _native

    lib = _native.load()
    assert b"sm_100a" in lib.hqmq_version()
    assert lib.hqmq_status_string(0) == b"ok"
    assert lib.hqmq_status_string(1) == b"invalid argument"
    assert lib.hqmq_pack_workspace_bytes(1000) >= 8000


def test_struct_layouts_match_header():
    """ctypes mirrors of the C structs have the C layout (sizes from the header order)."""
    from paper_2605_27646_b200 import _native

    assert ctypes.sizeof(_native.EncodeArgs) == 224
    assert _native.EncodeArgs.outlier_multiplier.offset == 48
    assert _native.EncodeArgs.data.offset == 64
    assert ctypes.sizeof(_native.DecodeArgs) == 152
    assert ctypes.sizeof(_native.PackedView) == 72
    assert _native.AttentionArgs.q.offset == 72


def test_c_struct_sizes_with_compiler(tmp_path):
    """Compile a probe against the header with gcc and compare struct layouts."""
    from paper_2605_27646_b200 import _native

    src = tmp_path / "probe.c"
    src.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "hqmq_b200.h"\n'
        "int main(){printf(\"%zu %zu %zu %zu %zu %zu\\n\", sizeof(hqmq_encode_args),"
        " sizeof(hqmq_decode_args), sizeof(hqmq_packed_view), sizeof(hqmq_attention_args),"
        " offsetof(hqmq_attention_args, workspace), offsetof(hqmq_encode_args, flag_capacity_words));"
        "return 0;}\n")
    exe = tmp_path / "probe"
    import subprocess

    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    out = [int(v) for v in subprocess.check_output([str(exe)]).split()]
    assert out == [ctypes.sizeof(_native.EncodeArgs), ctypes.sizeof(_native.DecodeArgs),
                   ctypes.sizeof(_native.PackedView), ctypes.sizeof(_native.AttentionArgs),
                   _native.AttentionArgs.workspace.offset,
                   _native.EncodeArgs.flag_capacity_words.offset]


def test_paged_struct_layouts_with_compiler(tmp_path):
    """The paged decode-attention structs (hqmq_paged_view / hqmq_paged_attention_args)."""
    from paper_2605_27646_b200 import _native

    src = tmp_path / "probe_paged.c"
    src.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "hqmq_b200.h"\n'
        "int main(){printf(\"%zu %zu %zu %zu %zu %zu\\n\", sizeof(hqmq_paged_view),"
        " sizeof(hqmq_paged_attention_args), offsetof(hqmq_paged_attention_args, scale),"
        " offsetof(hqmq_paged_attention_args, k), offsetof(hqmq_paged_attention_args, num_splits),"
        " offsetof(hqmq_paged_attention_args, workspace_bytes));return 0;}\n")
    exe = tmp_path / "probe_paged"
    import subprocess

    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    out = [int(v) for v in subprocess.check_output([str(exe)]).split()]
    A = _native.PagedAttentionArgs
    assert out == [ctypes.sizeof(_native.PagedView), ctypes.sizeof(A), A.scale.offset, A.k.offset,
                   A.num_splits.offset, A.workspace_bytes.offset]


def test_paged_append_struct_layout_with_compiler(tmp_path):
    """hqmq_paged_append_args as the C compiler lays it out."""
    from paper_2605_27646_b200 import _native

    src = tmp_path / "probe_append.c"
    src.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "hqmq_b200.h"\n'
        "int main(){printf(\"%zu %zu %zu %zu\\n\", sizeof(hqmq_paged_append_args),"
        " offsetof(hqmq_paged_append_args, num_pages), offsetof(hqmq_paged_append_args, src_index),"
        " offsetof(hqmq_paged_append_args, error_word));return 0;}\n")
    exe = tmp_path / "probe_append"
    import subprocess

    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    out = [int(v) for v in subprocess.check_output([str(exe)]).split()]
    A = _native.PagedAppendArgs
    assert out == [ctypes.sizeof(A), A.num_pages.offset, A.src_index.offset, A.error_word.offset]


def test_no_cpu_fallback_without_device():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    import numpy as np

    import paper_2605_27646_b200 as m

    with pytest.raises(m.NativeLibraryMissing):
        m.encode_tensor(np.zeros((1, 1, 4, 8)), m.CodecConfig(24, 3))
