cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/ab1_tests.log 2>&1; echo tests rc=$?
bash tools/ab_bench.sh > gpurun_out/ab1_ab.log 2>&1
bash tools/ab_bench.sh >> gpurun_out/ab1_ab.log 2>&1
timeout 300 python tools/phase_timing.py > gpurun_out/ab1_phase_new.log 2>&1
cp build/base_phase.sox paper_1911_01234_b200/libvdamp_b200_phase.so
timeout 300 python tools/phase_timing.py > gpurun_out/ab1_phase_base.log 2>&1
cat gpurun_out/ab1_ab.log
