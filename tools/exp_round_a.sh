# experiments batch A: pipe probes, NUMA H2D probe, cold setup per-stage, NTT prime-range chunking A/B
cd $GRAFT_REPO_ROOT
o=gpurun_out
./tools/probes/pipe_probes > $o/a_pipe_probes.txt 2>&1
timeout 300 python tools/h2d_numa_probe.py > $o/a_h2d_numa.txt 2>&1
(nproc; lscpu | grep -i -E "numa|model name|socket|^cpu\(s\)"; nvidia-smi topo -m) > $o/a_topo.txt 2>&1
timeout 600 python tools/setup_cold.py --busy > $o/a_setup_cold.txt 2>&1
for mb in 0 24 40 64; do
  echo "HG_NTT_L2_MB=$mb" >> $o/a_ntt_chunk.txt
  HG_NTT_L2_MB=$mb timeout 300 python tools/ntt_bench.py --variants 0 0 --rows-per-prime 4 --primes 105 >> $o/a_ntt_chunk.txt 2>&1
done
HG_NTT_L2_MB=40 timeout 900 python -m pytest -x -q tests/test_gpu_ring.py tests/test_gpu_fused.py tests/test_gpu_scale_parity.py > $o/a_chunk_tests.log 2>&1
echo "chunk tests rc=$?" >> $o/a_ntt_chunk.txt
for rep in 1 2; do
for mb in 0 32 48 80; do
  HG_NTT_L2_MB=$mb timeout 400 python bench.py --steps 5 --warmup 3 --no-e2e --no-primitives --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['kernel_classes']; print('L2_MB=$mb', d['value'], d['ms_per_step'], {c: k[c]['ms_per_step'] for c in k}, d['clocks'])" >> $o/a_ntt_chunk.txt 2>&1
done
done
