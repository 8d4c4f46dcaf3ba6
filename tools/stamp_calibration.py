import ctypes, sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2511_18296_b200 import _lib
lib = _lib.load(sys.argv[1]); _lib._lib = lib
lib.pp_debug_stamp.argtypes = [ctypes.c_void_p, ctypes.c_int]; lib.pp_debug_stamps.argtypes = [ctypes.c_void_p]
st = torch.cuda.Stream(); sp = st.cuda_stream
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
for rep in range(5):
    with torch.cuda.stream(st):
        flush.fill_(rep)
    lib.pp_debug_stamp(sp, 0); lib.pp_debug_stamp(sp, 1); lib.pp_debug_stamp(sp, 2); lib.pp_debug_stamp(sp, 3)
    st.synchronize()
s = np.zeros(8, np.uint64); lib.pp_debug_stamps(s.ctypes.data); s = s.astype(np.int64)
print("stamp gaps (us):", np.diff(s[:4]) / 1000)
