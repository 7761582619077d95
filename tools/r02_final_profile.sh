#!/bin/bash
# Final-build evidence: ncu --set full of the dominant kernel (E in residual mode) and the level-1
# V-cycle legs at the c4_weak_2049 sizes (helm_bench_graph regions: plain graphs, so ncu sees each
# kernel node), and the launch list of a host-polled bench-method solve (2 + 1 outer iterations).
set -u
mkdir -p gpurun_out
P='{"sstep": 8, "sstep_passes": 1, "inner_maxit": 192, "inner_restart": 48}'
NCU="ncu --set full --clock-control none --import-source on"
$NCU -k regex:k_glk_stream -c 1 -f -o gpurun_out/ncu_c4_glk_res_final python tools/ncu_regions.py --workload c4_weak_2049 --region ss_e --col 0 --params "$P" > gpurun_out/ncu_e.log 2>&1
$NCU -k regex:k_vc_down -c 1 -f -o gpurun_out/ncu_c4_vc_down1_final python tools/ncu_regions.py --workload c4_weak_2049 --region vc_down --col 1 --params "$P" > gpurun_out/ncu_down.log 2>&1
$NCU -k regex:k_vc_up -c 1 -f -o gpurun_out/ncu_c4_vc_up1_final python tools/ncu_regions.py --workload c4_weak_2049 --region vc_up --col 1 --params "$P" > gpurun_out/ncu_up.log 2>&1
$NCU -c 13 -f -o gpurun_out/ncu_c4_vcycle1_final python tools/ncu_regions.py --workload c4_weak_2049 --region vcycle --col 1 --params "$P" > gpurun_out/ncu_vc.log 2>&1
for r in glk_res vc_down1 vc_up1 vcycle1; do
  ncu -i gpurun_out/ncu_c4_${r}_final.ncu-rep --page raw --csv 2>/dev/null | gzip > gpurun_out/r02_final_ncu_c4_${r}_raw.csv.gz
done
ncu -i gpurun_out/ncu_c4_glk_res_final.ncu-rep --page source --csv 2>/dev/null | gzip > gpurun_out/r02_final_ncu_c4_glk_res_source.csv.gz
ls -la gpurun_out/*.ncu-rep
rm -f gpurun_out/*.ncu-rep   # gpurun_out is capped at 64 MiB: the raw / source pages travel back
PROBE_GRAPH=0 PROBE_MAXIT=1 PROBE_CAP=192 PROBE_M=48 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_c4_final.csv python tools/sstep_probe.py c4_weak_2049 8:1 > gpurun_out/launches_c4_final.log 2>&1
python tools/launch_summary.py gpurun_out/launches_c4_final.csv > gpurun_out/r02_launches_c4_final_summary.txt 2>&1
gzip -f gpurun_out/launches_c4_final.csv
head -12 gpurun_out/r02_launches_c4_final_summary.txt
