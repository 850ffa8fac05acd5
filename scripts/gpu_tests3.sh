python -m pytest tests/test_gpu_sense_model.py -q -rf -p no:cacheprovider -x 2>&1 | tail -15
