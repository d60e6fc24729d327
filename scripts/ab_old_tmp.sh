cd ab_old && python -m paper_2409_00657_b200.build > ../gpurun_out/ab_old_build.log 2>&1; cd ..
for r in 3 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2961$r bench.py --gpus 2 --no-model-centric > gpurun_out/ab_new_n2_$r.json 2> gpurun_out/ab_new_n2_$r.err
  (cd ab_old && timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2960$r bench.py --gpus 2 --no-model-centric > ../gpurun_out/ab_old_n2_$r.json 2> ../gpurun_out/ab_old_n2_$r.err)
done
python bench.py --no-cpu > gpurun_out/ab_new_n1.json 2> gpurun_out/ab_new_n1.err
(cd ab_old && python bench.py --no-cpu > ../gpurun_out/ab_old_n1.json 2> ../gpurun_out/ab_old_n1.err)
