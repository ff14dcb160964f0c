WS_LIBWS=paper_2408_00930_b200/lib/exp128/libws.so python tools/one.py cartpole 10000 0 1000 3 > gpurun_out/r02e_dbg.log 2>&1
tail -5 gpurun_out/r02e_dbg.log
