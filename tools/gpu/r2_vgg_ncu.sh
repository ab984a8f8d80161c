mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/vgg_launches.csv python tools/vgg_epoch_once.py 8 4 64 8 > gpurun_out/vgg_ncu.log 2>&1
tail -2 gpurun_out/vgg_ncu.log; wc -l gpurun_out/vgg_launches.csv
