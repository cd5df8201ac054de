timeout 1200 python -m pytest tests -q -m gpu 2>&1 | tail -6 > gpurun_out/f16_tests.log
DOGBLOB_CONV=umma DOGBLOB_STREAMED_UPLOAD=0 timeout 1200 python -m pytest tests -q -m gpu 2>&1 | tail -6 >> gpurun_out/f16_tests.log
python tools/config_timings.py 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: c=json.loads(l)
    except Exception: print(l[:150]); continue
    print(c['config'], 'lat', round(c['latency_ms_median'],3), 'conv', round(c['convolve_ms'],3), 'ext', round(c['extrema_ms'],3), 'prune', round(c['prune_ms'],3), 'blobs', c['blobs'])
" >> gpurun_out/f16_tests.log
python bench.py 2>/dev/null | python -c "
import sys, json
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('bench value', d['value'], 'e2e', d['e2e']['value'], 'lat', d['latency_ms']['single_frame_e2e_median'], d['latency_ms']['device_stage_ms_isolated'], 'frac', d['roofline']['frac'])
" >> gpurun_out/f16_tests.log
