python tools/ncu_decode.py > gpurun_out/ncu_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:decode_persistent -s 1 -c 1 \
    -o gpurun_out/pk_full python tools/ncu_decode.py > gpurun_out/ncu_run.log 2>&1
echo rc=$?; tail -3 gpurun_out/ncu_run.log; ls -la gpurun_out/
