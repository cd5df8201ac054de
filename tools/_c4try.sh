rm -f gpurun_out/variants.log
for s in 1 0; do
  echo "=== streamed=$s" >> gpurun_out/variants.log
  DOGBLOB_STREAMED_UPLOAD=$s python tools/config_timings.py C1 C2 C4 C5 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: c=json.loads(l)
    except Exception: print(l[:150]); continue
    print(c['config'], 'lat', round(c['latency_ms_median'],3), 'p90', round(c['latency_ms_p90'],3), 'conv', round(c['convolve_ms'],3))
" >> gpurun_out/variants.log
done
