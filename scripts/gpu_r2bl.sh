AB_LIB=paper_2209_02341_b200/lib/ab/qtrace.so ENERGON_ATTN_TRACE=gpurun_out/qt.txt timeout 300 python scripts/attn_qtrace.py
