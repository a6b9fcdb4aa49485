import ctypes, torch, sys
lib = ctypes.CDLL("paper_2411_17164_b200/libxmgn.so")
lib.xmgn_selftest_gemm.argtypes = [ctypes.c_int]*5 + [ctypes.c_void_p]*4
lib.xmgn_last_error.restype = ctypes.c_char_p
torch.manual_seed(0)
ok = True
for (M, N, K) in [(256, 128, 128), (300, 256, 512), (128, 64, 64)]:
    for amn in (0, 1):
        for bmn in (0, 1):
            A = torch.randn(M, K, device="cuda").bfloat16()
            B = torch.randn(N, K, device="cuda").bfloat16()
            Ain = A.t().contiguous() if amn else A
            Bin = B.t().contiguous() if bmn else B
            C = torch.zeros(M, N, device="cuda")
            st = lib.xmgn_selftest_gemm(M, N, K, amn, bmn, Ain.data_ptr(), Bin.data_ptr(), C.data_ptr(), None)
            torch.cuda.synchronize()
            ref = A.float() @ B.float().t()
            err = (C - ref).abs().max().item()
            print(M, N, K, amn, bmn, "status", st, lib.xmgn_last_error(), "maxerr", err, flush=True)
            ok &= (st == 0 and err < 1e-2)
print("ALL_OK" if ok else "FAIL")
