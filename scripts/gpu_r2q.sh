# MLP-down (TP=1) DRAM traffic vs schedule: stream-K tail on/off, A-panel group budget (ncu, one launch each)
mkdir -p gpurun_out
run() {
  tag=$1; shift
  env "$@" timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gemm_tc2 -s 5 -c 1 --csv python scripts/gemm_one.py 4096 5120 20480 0 2>/dev/null | python -c "
import sys, csv
rows=list(csv.reader(sys.stdin)); h=[i for i,r in enumerate(rows) if 'Metric Name' in r][0]; hdr=rows[h]
vals={r[hdr.index('Metric Name')]: (r[hdr.index('Metric Value')], r[hdr.index('Metric Unit')]) for r in rows[h+1:]}
print('$tag', vals)"
  echo "$tag timing: $(env "$@" timeout 60 python scripts/gemm_one.py 4096 5120 20480 0)"
}
run default X=1
run dp ENERGON_NO_STREAMK=1
run g48 ENERGON_GROUP_MB=48
run g130 ENERGON_GROUP_MB=130
run g200 ENERGON_GROUP_MB=200
run dp_g48 ENERGON_NO_STREAMK=1 ENERGON_GROUP_MB=48
run dp_g200 ENERGON_NO_STREAMK=1 ENERGON_GROUP_MB=200
