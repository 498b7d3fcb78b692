GNPC_LIB=$PWD/var/base.so python tools/flush_check.py gpurun_out/g16.npy
GNPC_LIB=$PWD/var/f64.so python tools/flush_check.py gpurun_out/g64.npy
