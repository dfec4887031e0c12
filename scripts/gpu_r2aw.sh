mkdir -p gpurun_out
python scripts/probe/cublas_shapes.py
timeout 300 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__cluster_dim_x,launch__cluster_dim_y,launch__block_size,launch__shared_mem_per_block_dynamic,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,dram__bytes_read.sum --csv python scripts/probe/cublas_shapes.py > gpurun_out/cublas_ncu.csv 2>&1
python - <<'P'
import csv
rows=[r for r in csv.reader(open('gpurun_out/cublas_ncu.csv')) if len(r)>10]
hdr=rows[0]; ki=hdr.index('Kernel Name'); mi=hdr.index('Metric Name'); vi=hdr.index('Metric Value'); ii=hdr.index('ID')
seen={}
for r in rows[1:]:
    seen.setdefault((r[ii], r[ki][:90]), {})[r[mi]]=r[vi]
import itertools
for (i,k),m in list(seen.items())[-8:]:
    print(i,k); print('   ',m)
P
for s in "4096 1920 5120 1" "4096 2560 5120 2" "4096 5120 640 0" "4096 5120 2560 0"; do python scripts/gemm_one.py $s; done
timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,dram__bytes_read.sum -c 6 --csv python scripts/gemm_one.py 4096 1920 5120 1 > gpurun_out/energon_qkv8_ncu.csv 2>&1; tail -12 gpurun_out/energon_qkv8_ncu.csv
