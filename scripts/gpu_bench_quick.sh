python -c "
from paper_2603_15042_b200 import _abi
print('ffma TF/s', _abi.measure_ffma_peak(0))
"
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
python -c "
import json
d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1])
print(d['value'], d['train_tflops'], d['timeslice'], d['tpot_distribution_ms'], d['config1']['roofline'], d['solo'], d['clocks'])
"
