# round-2 batch 5: tuner with the measured SimulateFn (1 part + folded K1
# forms; 2/8 logical parts through the measured MultiGpuReport), configs[4]
# sweep at 8 parts (auto and fine fetch), b200 profile re-fit from the probes
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2b5; mkdir -p $O
timeout 1500 python tools/tune_b200.py --workload products-gcn --exhaustive --fold-forms > $O/tune_products-gcn.json 2> $O/tune_products-gcn.err; tail -c 300 $O/tune_products-gcn.json
timeout 900 python tools/tune_b200.py --workload reddit-gcn --exhaustive > $O/tune_reddit-gcn.json 2> $O/tune_reddit-gcn.err; tail -c 300 $O/tune_reddit-gcn.json
timeout 900 python tools/tune_b200.py --workload products-gcn --parts 8 > $O/tune_products-gcn_8parts.json 2> $O/tune_p8.err; tail -c 300 $O/tune_products-gcn_8parts.json
timeout 900 python tools/tune_b200.py --workload config1 --parts 2 --exhaustive > $O/tune_config1_2parts.json 2> $O/tune_c1.err; tail -c 300 $O/tune_config1_2parts.json
timeout 2400 python tools/sweep_cfg5.py --parts 8 > $O/cfg5_sweep_auto.jsonl 2> $O/cfg5_auto.err; cut -c1-300 $O/cfg5_sweep_auto.jsonl
timeout 1800 python tools/sweep_cfg5.py --parts 8 --fetch fine --dims 16,64,256 > $O/cfg5_sweep_fine.jsonl 2> $O/cfg5_fine.err; cut -c1-300 $O/cfg5_sweep_fine.jsonl
timeout 600 python tools/refit_b200.py --out $O/refit.json > /dev/null 2> $O/refit.err; tail -c 600 $O/refit.json
