# Round evidence: the launch list of one ResNet-34 verification (image 1
# alone) and an ncu --set full capture of the conv kernel inside the 237-row
# pass (summarised on the box; the report travels back if small enough).
# usage (via gpurun): bash scripts/gpu/ncu_final.sh TAG
TAG=${1:-final}
mkdir -p gpurun_out
ONE_IMAGE_FIRST=1 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv python scripts/one_image.py cifar_resnet34 1 > gpurun_out/launches_$TAG.log 2>&1
tail -1 gpurun_out/launches_$TAG.log
python scripts/launch_summary.py gpurun_out/launches_$TAG.csv > gpurun_out/launches_$TAG.txt 2>&1
rm -f gpurun_out/launches_$TAG.csv
bash scripts/gpu/ncu_flat.sh $TAG 37 10 6
