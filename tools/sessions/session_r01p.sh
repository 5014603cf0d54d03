#!/bin/bash
tools/gpu_session.sh r01p tests
AB_TRIALS=10000000 tools/ab_session.sh r01p u1 win512 win8k win1m
