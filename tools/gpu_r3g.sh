#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_chain.py tests/test_gpu_parity.py -x -q -k "drelu or chain" 2>&1 | tail -2
timeout 300 python tools/drelu_ab.py > gpurun_out/drelu_ab5.json 2>&1; echo ab=$?; cat gpurun_out/drelu_ab5.json
prof() {
DR_NO_GRAPH=1 timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$2" -s $3 -c 1 -o /tmp/$1 python tools/c5_step.py 1 > gpurun_out/ncu_$1.log 2>&1; echo ncu=$?
ncu -i /tmp/$1.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$1.csv 2>/dev/null
ncu -i /tmp/$1.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/mix_$1.csv 2>/dev/null
python profiles/line_hot.py gpurun_out/mix_$1.csv 30
}
prof head 'tc2_rows_kernel<\(int\)-1>' 0
prof dz0 'tc2_rows_kernel<\(int\)0>' 0
