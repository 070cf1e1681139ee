for i in 1 2 3; do TC_ONLY_TIME=1 python tools/tc_check.py 2>&1 | tail -1; done > gpurun_out/tc.txt
cp tmp_libs/trace.so paper_2310_05218_b200/libslideconv_b200.so; python tools/tc_trace.py > gpurun_out/trace.txt 2>&1
