O=gpurun_out
PQTG_PHASES=1 PQTG_SPLIT=1 timeout 300 python tools/phase_probe.py sift1m 1 >> $O/pp3.txt 2>>$O/pp3_err.txt
PQTG_PHASES=1 PQTG_SPLIT=1 timeout 300 python tools/phase_probe.py sift1m 10 >> $O/pp3.txt 2>>$O/pp3_err.txt
PQTG_PHASES=1 PQTG_SPLIT=1 timeout 300 python tools/phase_probe.py deep100m 1 >> $O/pp3.txt 2>>$O/pp3_err.txt
