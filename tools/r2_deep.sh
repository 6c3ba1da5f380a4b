timeout 600 python benchmarks/gemm.py 204 512 768 1024 2048 > gpurun_out/r2j_gemm_base.jsonl 2>&1
CORTEX_LIB=variants/libcortex_deep.so timeout 600 python benchmarks/gemm.py 204 512 768 1024 2048 > gpurun_out/r2j_gemm_deep.jsonl 2>&1
python - <<'PY'
import json
b=[json.loads(l) for l in open('gpurun_out/r2j_gemm_base.jsonl') if l.startswith('{')]
d=[json.loads(l) for l in open('gpurun_out/r2j_gemm_deep.jsonl') if l.startswith('{')]
for x,y in zip(b,d):
    print(f"M={x['M']:5d} {x['name']:8s} base {x['ms']*1e3:7.1f} us deep {y['ms']*1e3:7.1f} us  ({y['ms']/x['ms']:.3f})")
PY
