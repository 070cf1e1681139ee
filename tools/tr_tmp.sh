cp tmp_libs/trace.so paper_2310_05218_b200/libslideconv_b200.so; python tools/tc_trace.py > gpurun_out/trace.txt 2>&1
