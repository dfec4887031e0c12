mkdir -p gpurun_out
AB_LIB=paper_2209_02341_b200/lib/ab/trace2.so ENERGON_ATTN_TRACE=gpurun_out/a2t_gpt3.txt CASE=gpt3 timeout 300 python scripts/attn_trace2.py > gpurun_out/a2t_gpt3_report.txt 2>&1; head -70 gpurun_out/a2t_gpt3_report.txt
AB_LIB=paper_2209_02341_b200/lib/ab/trace2.so ENERGON_ATTN_TRACE=gpurun_out/a2t_s2048.txt CASE=s2048 timeout 300 python scripts/attn_trace2.py > gpurun_out/a2t_s2048_report.txt 2>&1; head -40 gpurun_out/a2t_s2048_report.txt
