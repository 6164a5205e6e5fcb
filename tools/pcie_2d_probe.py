"""PCIe probe for a column-panelled host pipeline: pinned D2H / H2D of a
row-major M x N fp32 matrix as column panels (cudaMemcpy2DAsync: width w*4
bytes, pitch N*4) vs one contiguous copy.  Prints one JSON line per case."""
import ctypes
import json
import time

import torch

cudart = ctypes.CDLL("libcudart.so")
cudart.cudaMemcpy2DAsync.restype = ctypes.c_int
cudart.cudaMemcpy2DAsync.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_size_t,
                                     ctypes.c_size_t, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
D2H, H2D = 2, 1


def main():
    dev = torch.device("cuda:0")
    M, N = 1 << 20, 64
    d = torch.empty((M, N), device=dev)
    h = torch.empty((M, N), pin_memory=True)
    s = torch.cuda.current_stream(dev)
    for kind, name in ((D2H, "D2H"), (H2D, "H2D")):
        for w in (64, 32, 16, 8):
            best = 1e9
            for _ in range(5):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                for c0 in range(0, N, w):
                    if kind == D2H:
                        rc = cudart.cudaMemcpy2DAsync(h.data_ptr() + 4 * c0, N * 4, d.data_ptr() + 4 * c0, N * 4,
                                                      w * 4, M, D2H, s.cuda_stream)
                    else:
                        rc = cudart.cudaMemcpy2DAsync(d.data_ptr() + 4 * c0, N * 4, h.data_ptr() + 4 * c0, N * 4,
                                                      w * 4, M, H2D, s.cuda_stream)
                    assert rc == 0, rc
                torch.cuda.synchronize()
                best = min(best, time.perf_counter() - t0)
            print(json.dumps({"dir": name, "M": M, "N": N, "panel_cols": w, "piece_bytes": 4 * w,
                              "ms": round(best * 1e3, 3), "GBs": round(M * N * 4 / best / 1e9, 1)}), flush=True)


if __name__ == "__main__":
    main()
