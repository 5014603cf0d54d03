#!/bin/bash
tools/gpu_session.sh r01q tests
tools/all_configs.sh r01q
tools/gpu_session.sh r01q ncu
