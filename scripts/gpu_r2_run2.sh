mkdir -p gpurun_out/m22
for i in 1 2 3 4; do
timeout 900 python -X faulthandler -m pytest tests -m gpu -q -s -p no:cacheprovider > gpurun_out/m22/pytest_full_$i.txt 2>&1
echo "run $i rc=$?"
grep -n -A30 "Fatal Python" gpurun_out/m22/pytest_full_$i.txt | head -45
grep -E "^FAILED|^E  " gpurun_out/m22/pytest_full_$i.txt | head -5
tail -1 gpurun_out/m22/pytest_full_$i.txt
done
