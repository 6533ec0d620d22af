# Warp-stall sampling of the persistent attention kernel (Cog with the decoupled-P build, Wan) + full GPU suite on the decoupled-P build
mkdir -p gpurun_out/r02stall
P=gpurun_out/r02stall
L="libblade_asa_BLADE_ATTN2P_SEPP=1.so"
BLADE_LIB=$L ncu --set full --import-source on --clock-control none -k regex:attn_tc2p -s 3 -c 1 -o $P/cog_sepp -f python scripts/attn_time.py --workload cog --calls 2 --blocks 1 > $P/ncu_cog.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:attn_tc2p -s 3 -c 1 -o $P/wan -f python scripts/attn_time.py --workload wan --calls 2 --blocks 1 > $P/ncu_wan.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:probe2 -s 1 -c 1 -o $P/probe_wan -f python scripts/mask_time.py --workload wan --configs keep51 --steps 2 > $P/ncu_probe.log 2>&1
BLADE_LIB=$L timeout 1500 python -m pytest tests -m gpu -q -x > $P/pytest_sepp.log 2>&1; echo "rc=$?" >> $P/pytest_sepp.log
tail -3 $P/pytest_sepp.log; ls -la $P
