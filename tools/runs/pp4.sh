O=gpurun_out
PQTG_PHASES=1 timeout 300 python tools/phase_probe.py sift1m 1 >> $O/pp4.txt 2>>$O/pp4_err.txt
