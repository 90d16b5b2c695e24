"""Print the device's L2 size and persisting-L2 limits (development tool)."""
import torch
from cuda.bindings import runtime as rt
err, p = rt.cudaGetDeviceProperties(0)
print("l2CacheSize", p.l2CacheSize, "persistingL2CacheMaxSize", p.persistingL2CacheMaxSize,
      "accessPolicyMaxWindowSize", p.accessPolicyMaxWindowSize)
