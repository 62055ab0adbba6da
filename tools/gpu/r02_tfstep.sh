set -x
timeout 900 python -m pytest tests/test_gpu_step_config.py -m gpu -q -k tf_step > gpurun_out/r02_tfstep.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/r02_tfstep.log
(cd tests && timeout 900 python parity_report.py) > gpurun_out/r02_parity2.json 2> gpurun_out/r02_parity2.err; echo "parity rc=$?"; tail -3 gpurun_out/r02_parity2.err
python -c "import json;d=json.load(open('gpurun_out/r02_parity2.json'));print(json.dumps(d['worst']));print({k:v for k,v in d['cases'].items() if k.startswith(('C1_step','C2_step'))})"
