#!/bin/bash
# tensor-core column pass v2 (tools/exp/tc1): parity subset, then A/B against the butterfly build
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/r2c
HKS_LIB_PATH=tools/exp/tc1/libhks.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider \
  -k "ntt_parity or keyswitch_parity or hmult or rotate or linear_transform or moddown or modup or rescale or concurrent" > ${O}_pytest.txt 2>&1
echo "pytest rc=$?" >> ${O}_pytest.txt
timeout 600 bash tools/ab.sh r2c tc1
python -c "import torch; p=torch.cuda.get_device_properties(0); print(p)" > ${O}_props.txt 2>&1
python - >> ${O}_props.txt 2>&1 <<'PY'
import ctypes
rt = ctypes.CDLL("libcudart.so")
for name, attr in (("MaxPersistingL2CacheSize", 108), ("MaxAccessPolicyWindowSize", 109), ("L2CacheSize", 38)):
    v = ctypes.c_int()
    rt.cudaDeviceGetAttribute(ctypes.byref(v), attr, 0)
    print(name, v.value)
PY
