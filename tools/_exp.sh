P="python tools/phase_times.py"
for lib in "" paper_1704_07355_b200/_lib/old/libqadc_b200.so paper_1704_07355_b200/_lib/n512/libqadc_b200.so; do
echo "lib=$lib"
QADC_B200_LIB=$lib $P cfg1 2>&1 | grep -E "k_select"
QADC_B200_LIB=$lib $P cfg2 30000000 10000 2>&1 | grep -E "k_select"
done
