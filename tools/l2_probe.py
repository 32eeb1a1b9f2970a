"""Print the B200's L2 persistence limits (cudaDevAttrMaxPersistingL2CacheSize,
cudaDevAttrMaxAccessPolicyWindowSize, L2 size)."""
from cuda.bindings import runtime as rt

for name in ("cudaDevAttrL2CacheSize", "cudaDevAttrMaxPersistingL2CacheSize",
             "cudaDevAttrMaxAccessPolicyWindowSize"):
    err, v = rt.cudaDeviceGetAttribute(getattr(rt.cudaDeviceAttr, name), 0)
    print(name, err, v)
