timeout 200 python tools/umma_debug.py C1 2>&1 | grep "umma\]\|blob sets" | cut -c1-220 > gpurun_out/variants.log
timeout 200 python tools/umma_debug.py C2 2>&1 | grep "umma\]\|blob sets" | cut -c1-220 >> gpurun_out/variants.log
UMMA_PROF_MASKS=0 timeout 200 python tools/umma_probe.py C2 >> gpurun_out/variants.log 2>&1
timeout 300 python tools/umma_probe.py C4 2>&1 | grep "^umma  .*row" >> gpurun_out/variants.log
timeout 1200 python -m pytest tests -q -m gpu 2>&1 | tail -8 >> gpurun_out/variants.log
