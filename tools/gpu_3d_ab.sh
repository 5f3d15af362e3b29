# 3-D A/B: default libmandel3d.so vs a variant built with -D$DEF (MANDEL3D_LIB), bench3d + parity.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python tools/bench3d.py V1 V2 | python -c "
import json,sys
for l in sys.stdin: d=json.loads(l); print('default', d['config']['name'], round(d['ask_ms'],3))"
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -ftz=false -prec-div=true -prec-sqrt=true -Xcompiler -fPIC -shared -D$DEF -o /tmp/lib3v.so paper_2206_02255_b200/csrc/mandel3d.cu
MANDEL3D_LIB=/tmp/lib3v.so timeout 600 python tools/bench3d.py V1 V2 | python -c "
import json,sys
for l in sys.stdin: d=json.loads(l); print('$DEF', d['config']['name'], round(d['ask_ms'],3))"
MANDEL3D_LIB=/tmp/lib3v.so timeout 600 python -m pytest tests/test_gpu_3d.py -q -x 2>&1 | tail -1
