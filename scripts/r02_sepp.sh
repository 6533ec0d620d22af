# decoupled-P (kSepP) schedule of the persistent kernel for d = 64: parity, then interleaved timing
mkdir -p gpurun_out/r02sepp
P=gpurun_out/r02sepp
BLADE_LIB="libblade_asa_BLADE_ATTN2P_SEPP=1.so" timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py tests/test_gpu_gt.py -q -x > $P/pytest_sepp.log 2>&1; echo "rc=$?" >> $P/pytest_sepp.log
tail -3 $P/pytest_sepp.log
for rep in 1 2; do
for lib in libblade_asa.so "libblade_asa_BLADE_ATTN2P_SEPP=1.so" "libblade_asa_BLADE_ATTN2P_SEPP=1,BLADE_ATTN2P_EMU64=0x11.so" "libblade_asa_BLADE_ATTN2P_SEPP=1,BLADE_ATTN2P_EMU64=0x00.so"; do
  BLADE_LIB=$lib timeout 300 python scripts/attn_time.py --workload cog --calls 50 --blocks 3 >> $P/cog.jsonl 2>&1
done
done
cat $P/cog.jsonl
