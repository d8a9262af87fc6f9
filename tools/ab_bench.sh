for l in "" old "" old; do
  W4A16_LIB=$l timeout 400 python bench.py --steps 10 --warmup 3 --sweep "1,8,16" --no-kernels --no-lm-head --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$l' or 'main', round(d['value'],3), round(d['ms_per_step'],3), {k:round(v['TBps'],3) for k,v in d['m_sweep'].items()})"
done
