mkdir -p gpurun_out
O=gpurun_out/dbg7.txt
timeout 300 python tools/batch_check.py c4M f64 512 auto 512 >> $O 2>&1
timeout 300 python tools/batch_check.py c4M f64 512 materialized 512 >> $O 2>&1
timeout 300 python tools/batch_check.py c4M f64 2048 auto 4096 >> $O 2>&1
JT_OWN_MULTI=1 timeout 300 python tools/batch_check.py c4M f64 256 auto 512 >> $O 2>&1
JT_OWN_MULTI=1 timeout 300 python tools/batch_check.py c4M f64 512 auto 512 >> $O 2>&1
JT_OWN_MULTI=1 timeout 300 python tools/batch_check.py c5 f64 128 auto 256 >> $O 2>&1
echo "[OWN_MULTI tests]" >> $O
JT_OWN_MULTI=1 timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider >> $O 2>&1
echo "[single OWN_MULTI]" >> $O
JT_OWN_MULTI=1 timeout 300 python tools/single_bench.py c2 c4M c5 c4B >> $O 2>&1
