for v in "" "TT_MC_SPL=4" "TT_MC_WAVES=2" "TT_MC_WAVES=4" "TT_MC_SPL=4 TT_MC_WAVES=2"; do
  for n in 16 32; do
    env $v timeout 200 python bench.py --samples $n --sweep "" --no-cpu-baseline --steps 20 > gpurun_out/exp.json 2>/dev/null
    python -c "import json,sys;d=json.load(open('gpurun_out/exp.json'));print('$v', $n, round(d['roofline']['kernel_ms'],4), round(d['ms_per_step'],4))"
  done
done
