set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -15
timeout 600 python bench.py > gpurun_out/bench1.json 2> gpurun_out/bench1.err; tail -3 gpurun_out/bench1.err
cat gpurun_out/bench1.json
python -c "
import ctypes as C; l=C.CDLL('paper_2403_01596_b200/lib/libp2p_peaks.so'); 
for f in ['p2p_peak_mufu_lg2','p2p_peak_ffma2','p2p_peak_dfma','p2p_peak_hbm_read']:
    v=C.c_double(0); getattr(l,f).argtypes=[C.c_int,C.POINTER(C.c_double)]; r=getattr(l,f)(0,C.byref(v)); print(f, r, '%.4e'%v.value)
" | tee gpurun_out/peaks1.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches1.csv python bench.py --steps 2 --warmup 1 --profile > /dev/null 2>&1; tail -5 gpurun_out/launches1.csv
