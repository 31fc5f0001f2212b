set -x
mkdir -p gpurun_out/v4
timeout 300 python tools/pre_time.py C5 > gpurun_out/v4/pre_time_c5.txt 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rows -s 5 -c 1 -o gpurun_out/v4/prof_r02_pre_rows_c5 -f python tools/pre_time.py C5 > gpurun_out/v4/ncu_pre.log 2>&1
tail -2 gpurun_out/v4/ncu_pre.log
timeout 300 python tools/fapply_run.py C3 > gpurun_out/v4/fapply_c3.txt 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sym_stream -s 2 -c 1 -o gpurun_out/v4/prof_r02_sym_stream_c3 -f python tools/fapply_run.py C3 > gpurun_out/v4/ncu_sym.log 2>&1
tail -2 gpurun_out/v4/ncu_sym.log
ls -la gpurun_out/v4/*.ncu-rep
