"""A few eager launches of the nibble-operand (kind::mxf4) Boolean products,
for ncu: 8192^3 on the plain kernel, 1024^3 on the split-K pair, and 16
stacked 1024^3 products on the batched kernel."""
import sys; sys.path.insert(0, '.')
import torch
from paper_1705_08743_b200 import _native
lib = _native.lib(); lib.smx_set_graphs(0)
sp = _native.stream_ptr
for rows, n, batched in ((8192, 8192, 0), (1024, 1024, 0), (16 * 1024, 1024, 16)):
    A = (torch.rand((rows, n), device="cuda") < 0.05).to(torch.uint8)
    A4 = (A[:, 0::2] * 2 + A[:, 1::2] * 32).contiguous()
    C = torch.zeros((rows, n // 32), dtype=torch.int32, device="cuda")
    for _ in range(3):
        if batched:
            _native.check(lib.smx_bool_gemm_f4_batched(A4.data_ptr(), A4.data_ptr(), C.data_ptr(), batched, n, n, n,
                                                       n // 2, n // 2, n // 32, 0, sp()), "f4 batched")
        else:
            _native.check(lib.smx_bool_gemm_f4(A4.data_ptr(), A4.data_ptr(), C.data_ptr(), n, n, n, n // 2, n // 2,
                                               n // 32, 0, sp()), "f4")
    torch.cuda.synchronize()
