# decode context-split variants: private_us / GB/s of one config-2 layer's private contexts
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 1 2; do
for lib in "" variants/st3.so variants/st4.so variants/sp16.so variants/nocomp.so; do
  for sc in 1 2; do
    CORTEX_LIB=$lib CORTEX_PRIV_SCALE=$sc timeout 300 python benchmarks/attn_step.py --private-only
  done
done
done
for lib in variants/base.so variants/g2nofeedx.so variants/g2nofeed.so; do
  echo "== $lib"
  CORTEX_LIB=$lib timeout 300 python benchmarks/gemm.py 512 768 1536 2>&1 | grep '^{' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['M'],d['name'],round(d['ms']*1e3,1),'us',round(d['tflops']),'TF/s',d['tile2'])"
done
