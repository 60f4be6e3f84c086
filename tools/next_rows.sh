#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/b.log 2>&1
timeout 600 python -m pytest tests/test_gpu_next.py tests/test_gpu_parity.py -x -q -k "kprofile or sweep or sum_merge" > gpurun_out/t.log 2>&1; tail -3 gpurun_out/t.log
timeout 600 python tools/breakdown.py C5 > gpurun_out/breakdown_c5.json 2> gpurun_out/breakdown_c5.err; cat gpurun_out/breakdown_c5.json; tail -2 gpurun_out/breakdown_c5.err
timeout 600 python tools/breakdown.py C2 > gpurun_out/breakdown_c2.json 2> gpurun_out/breakdown_c2.err; cat gpurun_out/breakdown_c2.json; tail -2 gpurun_out/breakdown_c2.err
timeout 900 python tools/ksweep.py C3 > gpurun_out/ksweep_c3.json 2> gpurun_out/ksweep_c3.err; cat gpurun_out/ksweep_c3.json; tail -2 gpurun_out/ksweep_c3.err
