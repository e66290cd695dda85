"""Runs the ctypes stub of INTEGRATION.md section 2 against the oracle scan (test infrastructure)."""
# hqmq/kernels.py — B200 backend for nearest_scan (_kernels.pyx:16-46)
import ctypes, numpy as np, torch
_lib = ctypes.CDLL("paper_2605_27646_b200/_lib/libhqmq_b200.so")
_lib.hqmq_nearest_scan.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                   ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                   ctypes.c_void_p]
_lib.hqmq_nearest_scan.restype = ctypes.c_int
_lib.hqmq_status_string.argtypes = [ctypes.c_int]
_lib.hqmq_status_string.restype = ctypes.c_char_p

def _nearest_scan_b200(dirs, codewords):
    d = torch.from_numpy(np.ascontiguousarray(dirs, np.float64)).cuda()
    c = torch.from_numpy(np.ascontiguousarray(codewords, np.float64)).cuda()
    idx = torch.empty(d.shape[0], dtype=torch.int64, device="cuda")
    cos = torch.empty(d.shape[0], dtype=torch.float64, device="cuda")
    st = _lib.hqmq_nearest_scan(d.data_ptr(), d.shape[0], c.data_ptr(), c.shape[0],
                                idx.data_ptr(), cos.data_ptr(),
                                ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    if st != 0:
        raise RuntimeError(_lib.hqmq_status_string(st).decode())
    return idx.cpu().numpy(), cos.cpu().numpy()

import sys
sys.path.insert(0, "oracle")
import hqmq_oracle as O
rs = np.random.default_rng(0)
d = rs.standard_normal((1000, 4)); d /= np.linalg.norm(d, axis=1, keepdims=True)
cw = np.ascontiguousarray(O.Bank(0, 64).joint(0, 0, "K").reshape(-1, 4))
idx, cos = _nearest_scan_b200(d, cw)
ridx, rcos = O.nearest_scan(d, cw)
print("stub matches oracle:", np.array_equal(idx, ridx), np.array_equal(cos, rcos))
