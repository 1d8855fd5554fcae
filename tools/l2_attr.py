"""Print the device's L2 / access-policy limits (cudaDeviceGetAttribute via ctypes)."""
import ctypes, glob, torch
torch.cuda.init()
lib = ctypes.CDLL(glob.glob("/usr/local/cuda/lib64/libcudart.so*")[0])
for name, attr in [("l2_bytes", 38), ("max_persisting_l2", 108), ("max_access_policy_window", 109)]:
    v = ctypes.c_int(0)
    rc = lib.cudaDeviceGetAttribute(ctypes.byref(v), attr, 0)
    print(name, rc, v.value)
