# split-k slice count sweep (KW_SPLITK_SLICES) on small-output / long-k shapes, config 27 vs the model's choice
mkdir -p gpurun_out
for shape in 512,512,16384 256,256,65536 1024,512,8192 768,768,8192 512,512,4096 512,512,2048 128,128,32768; do
  for S in 0 2 3 4 6 8 12 16 24 32; do
    KW_SPLITK_SLICES=$S timeout 120 python tools/dgemm_rect.py $shape 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$shape S=$S', 'cfg27', d['cfgs'].get('27'), 'lib', d['library'], 'cublas', d['cublas'])"
  done
done
