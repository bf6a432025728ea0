# ncu --set full of the run-strip kernel (one launch): CFG, NS, NQ, LIB, TAG env
set -x
CFG=${CFG:-C5a}; TAG=${TAG:-x}
export PM_TMA_NS=${NS:-2} PM_TMA_NQ=${NQ:-2} PM_NATIVE_LIB=$LIB
timeout 120 python tools/one_apply.py $CFG striptma 2 && \
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_strip_tma -s 1 -c 1 \
   -o gpurun_out/prof_tma_${CFG}_$TAG -f python tools/one_apply.py $CFG striptma 2 > gpurun_out/ncu_tma_$TAG.log 2>&1
python tools/ncu_brief.py gpurun_out/prof_tma_${CFG}_$TAG.ncu-rep | tee gpurun_out/brief_tma_${CFG}_$TAG.txt
