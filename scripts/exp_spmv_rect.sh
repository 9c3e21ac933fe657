# C5 folded-R SpMV: lanes per row sweep (TT_SPMV_RECT_LPR), kernel time and step time
for v in ${LPRS:-4 8 16 32}; do
  TT_SPMV_RECT_LPR=$v timeout 300 python bench.py --config c5 --sweep "" --no-cpu-baseline --steps 30 > gpurun_out/exp.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/exp.json'));print('LPR=$v', round(d['roofline']['kernel_ms']*1e3,1), 'us', round(d['roofline']['frac'],3), round(d['ms_per_step'],4), 'ms/step')"
done
