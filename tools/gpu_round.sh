#!/bin/bash
# One GPU pass for the round's evidence (round 2): the GPU test suite and smoke(); bench lines (C4
# fp32/fp64 fused and split, the tcgen05 variant, C5, C5w, the dry multi-partition run, the reference
# arm, the 3D order sweep); the ncu launch list of the default bench; full ncu of the stage kernels
# (5 launches = one LSERK4 step) for C4 fp32, C4 fp64, split C4 fp32, C5 (N=8 fp64 material: the
# warp-specialised DMMA kernel) and the tcgen05 variant.
# The ncu captures run first so that the bench lines carry this build's DRAM traffic.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/gputest.log 2>&1; tail -1 gpurun_out/gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:stage_kernel -s 10 -c 5 -o gpurun_out/fused_n5_f32 \
    python tools/prof_one.py 5 4 724 1 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:stage_kernel -s 10 -c 5 -o gpurun_out/fused_n5_f64 \
    python tools/prof_one.py 5 8 724 1 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:stage_kernel -s 20 -c 10 -o gpurun_out/split_n5_f32 \
    python tools/prof_one.py 5 4 724 0 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:stage_kernel -s 10 -c 5 -o gpurun_out/fused_n8_f64_mat \
    python tools/prof_mat.py 8 8 1448 3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:stage_kernel_tc -s 10 -c 5 -o gpurun_out/tc_n5_f32 \
    python tools/prof_one.py 5 4 724 1 3 1 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/fused_n5_f32.ncu-rep gpurun_out/fused_n5_f64.ncu-rep \
    gpurun_out/split_n5_f32.ncu-rep gpurun_out/fused_n8_f64_mat.ncu-rep gpurun_out/tc_n5_f32.ncu-rep \
    > gpurun_out/ncu_summary.txt 2>&1
python tools/traffic.py N5_p4_n724_P1_fused=gpurun_out/fused_n5_f32.ncu-rep \
    N5_p8_n724_P1_fused=gpurun_out/fused_n5_f64.ncu-rep N5_p4_n724_P1_split=gpurun_out/split_n5_f32.ncu-rep \
    N8_p8_n1448_P1_fused=gpurun_out/fused_n8_f64_mat.ncu-rep > gpurun_out/traffic.log 2>&1
cp profiles/traffic.json gpurun_out/traffic.json  # the benches below read it (roofline.traffic)
ncu -i gpurun_out/fused_n5_f32.ncu-rep --page source --csv --print-source sass > gpurun_out/fused_n5_f32_sass.csv 2>&1
ncu -i gpurun_out/tc_n5_f32.ncu-rep --page source --csv --print-source sass > gpurun_out/tc_n5_f32_sass.csv 2>&1
rm -f gpurun_out/*.ncu-rep
python bench.py --steps 200 --warmup 10 > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --steps 200 --warmup 10 --prec 8 --no-cpu-baseline > gpurun_out/bench_f64.json 2>> gpurun_out/bench.err
python bench.py --steps 200 --warmup 10 --variant tcgen05 --no-cpu-baseline > gpurun_out/bench_tc.json 2>> gpurun_out/bench.err
python bench.py --split --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_split.json 2>> gpurun_out/bench.err
python bench.py --split --prec 8 --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_f64_split.json 2>> gpurun_out/bench.err
python bench.py --config c5 --steps 20 --warmup 3 --ref-n 16 --ref-steps 20 > gpurun_out/bench_c5.json 2>> gpurun_out/bench.err
python bench.py --config c5w --steps 40 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5w.json 2>> gpurun_out/bench.err
python bench.py --partitions 4 --steps 100 --warmup 5 > gpurun_out/bench_dry4.json 2>> gpurun_out/bench.err
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err
rm -f gpurun_out/bench3d.jsonl
for prec in 4 8; do for n in 1 2 3 4 5; do
  python bench.py --dim 3 --order $n --prec $prec --steps 20 --warmup 3 --no-cpu-baseline 2>> gpurun_out/bench.err | tail -1 >> gpurun_out/bench3d.jsonl
done; done
ls -la gpurun_out
