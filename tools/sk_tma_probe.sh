# split-K partials through the C ring (TK_SK_TMA) vs per-thread stores/loads: parity subset + timing (tuning)
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "split" 2>&1 | tail -2
TK_SK_TMA=0 timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "split" 2>&1 | tail -1
TK_SPLITK_MINKB=4 timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "split" 2>&1 | tail -1
export GRAPH=1
for cfg in "TK_SK_TMA=1" "TK_SK_TMA=0"; do
  env $cfg python -c "
import os,sys; sys.path.insert(0,'.')
import tools.bench_variants as bv
bv.dense(4096, m=1536, k=16384, name='split 1536x4096x16384 $cfg')
bv.dense(4096, m=4096, k=16384, name='split 4096x4096x16384 $cfg')
os.environ['TK_PAIR_BNI']='256'; os.environ['TK_SPLITK_MINKB']='4'
bv.dense(1024, name='1024^3 bni256 split4 $cfg')
os.environ['TK_SPLITK_MINKB']='8'
bv.dense(1024, name='1024^3 bni256 split2 $cfg')
os.environ['TK_PAIR_BNI']='128'
bv.dense(1024, name='1024^3 bni128 split2 $cfg')
os.environ['TK_PAIR_BNI']='64'; os.environ['TK_SPLITK_MINKB']='64'
bv.dense(1024, name='1024^3 bni64 nosplit $cfg')
" 2>&1 | grep TFLOPS | cut -c1-100
done
