"""cuBLAS DGEMM yardstick (torch.matmul fp64) on the K1/K2 shapes of SURVEY.md §8(d). Not product code."""
import json, torch
dev = torch.device("cuda:0")
for (M, N, K, name) in [(8192, 10000, 10000, "K1_C4"), (8192, 7000, 10000, "K2_C4"), (15104, 10000, 10000, "K1_C4_k15104"),
                        (15104, 7016, 10000, "K2_C4_k15104"), (8192, 1000, 1000, "K1_C1"), (8192, 6000, 1000, "K2_C2"),
                        (4736, 7016, 1000, "K2_C2_k4736"), (8192, 8192, 8192, "sq8192")]:
    a = torch.randn(M, K, dtype=torch.float64, device=dev)
    b = torch.randn(K, N, dtype=torch.float64, device=dev)
    for _ in range(3):
        c = a @ b
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); c = a @ b; e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(json.dumps({"gemm": name, "M": M, "N": N, "K": K, "ms": round(best, 3), "tflops": round(2 * M * N * K / best / 1e9, 2)}))
