import ctypes as C, torch
torch.cuda.init()
lib = C.CDLL("libcuda.so.1")
enc = lib.cuTensorMapEncodeTiled
enc.restype = C.c_int
buf = torch.zeros(1 << 20, dtype=torch.float64, device="cuda")
base = buf.data_ptr() + 4096
def try_map(rank, dims, strides, box):
    m = (C.c_ubyte * 128)()
    d = (C.c_uint64 * rank)(*dims)
    s = (C.c_uint64 * max(rank - 1, 1))(*(strides or [0]))
    b = (C.c_uint32 * rank)(*box)
    e = (C.c_uint32 * rank)(*([1] * rank))
    # dtype FLOAT64 = 8? enumerate: UINT8=0,UINT16,UINT32,INT32,UINT64,INT64,FLOAT16,FLOAT32,FLOAT64=8
    r = enc(m, 8, rank, C.c_void_p(base), d, s if rank > 1 else None, b, e, 0, 0, 0, 0)
    return r
for n in (36, 37, 64, 65, 96, 97, 128, 129, 8192, 8193):
    for box in (20, 128):
        print("rank2 n=%d box=%d -> %d" % (n, box, try_map(2, [n, 1], [(n * 8 + 15) // 16 * 16], [box, 1])),
              " rank1 -> %d" % try_map(1, [n], None, [box]))
