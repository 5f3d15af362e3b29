set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
MANDEL_TRACE_DEFS=MANDEL_RFB_PACK=0,MANDEL_RF_MINB=4 timeout 300 python tools/trace_refill.py C3 --P 8 > gpurun_out/trace45.txt 2>&1; cat gpurun_out/trace45.txt | cut -c1-300
