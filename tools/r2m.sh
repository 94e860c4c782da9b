timeout 900 python -m pytest tests/test_gpu_pool.py tests/test_gpu_backbone.py tests/test_gpu_headline.py -q -p no:cacheprovider -x > gpurun_out/r2m_tests.log 2>&1; echo "exit $?" >> gpurun_out/r2m_tests.log
tail -3 gpurun_out/r2m_tests.log; grep -E "^E  |FAILED" gpurun_out/r2m_tests.log | head
timeout 300 python tools/psh_bench.py 2>&1 | tail -4
cat > /tmp/gemm_drive.py <<'PY'
import torch, sys
sys.path.insert(0, ".")
from paper_2412_16481_b200 import _lib as L
n, K, N = 1000, 96, 288
x = torch.randn(n, K, device="cuda").to(torch.bfloat16)
w = torch.randn(N, K, device="cuda").to(torch.bfloat16)
b = torch.randn(N, device="cuda")
y = torch.empty(n, N, device="cuda", dtype=torch.bfloat16)
L.call("f3d_gemm", L.ptr(x), K, n, K, L.ptr(w), N, L.ptr(b), 0, L.ptr(y), N, None, L.stream())
torch.cuda.synchronize(); print("gemm ok")
PY
timeout 300 compute-sanitizer --tool synccheck --print-limit 5 python /tmp/gemm_drive.py 2>&1 | grep -v "Host Frame" | head -30
