#!/bin/bash
# GPU box: full GPU tests, then bench lines (default + given configs) and the reference arm.
tag=${1:-run}; shift
mkdir -p gpurun_out
if [ -z "$NO_TESTS" ]; then
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_${tag}.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_${tag}.log
fi
for c in ${CONFIGS:-garden}; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-20} --warmup 5 > gpurun_out/bench_${tag}_$c.json 2> gpurun_out/bench_${tag}_$c.err
  echo "bench $c rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/bench_${tag}_$c.json').read().strip().splitlines()[-1]);print('$c fps',round(d['value'],1),'render-only',round(d['render_only_value'],1),'e2e',round(d.get('e2e',{}).get('value',0),1),'e2e1',round(d.get('e2e_frame_upload',{}).get('value',0),1),'rp',round(d.get('e2e_run_pipeline',{}).get('value',0),2),'res',round(d.get('e2e_resident',{}).get('value',0),1),'roof',round(d['roofline']['frac'],3),'bin',round(d['binning_roofline']['frac'],3),'clk',d['clocks'].get('sm_mhz'),d['clocks'].get('reasons'))" || tail -5 gpurun_out/bench_${tag}_$c.err
done
if [ -n "$REF" ]; then
  timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref_${tag}.json 2> gpurun_out/ref_${tag}.err
  echo "ref rc=$?"; tail -c 400 gpurun_out/ref_${tag}.json
fi
