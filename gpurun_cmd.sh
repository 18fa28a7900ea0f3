ls -la oracle/_ref/; nproc; lscpu | grep -i "model name\|^CPU(s)"
timeout 120 ./oracle/_ref/ref_driver bench-lsm mamba2 1 262144 16 128 64 0 10 ; echo rc=$?
